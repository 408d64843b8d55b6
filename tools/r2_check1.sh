# round 2 first GPU check: new full-size / cross-term tests, whole GPU suite, default bench
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -rA > gpurun_out/r2a/t_full.log 2>&1; echo "exit $?" >> gpurun_out/r2a/t_full.log
tail -5 gpurun_out/r2a/t_full.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullsize.py > gpurun_out/r2a/t_all.log 2>&1; echo "exit $?" >> gpurun_out/r2a/t_all.log
tail -5 gpurun_out/r2a/t_all.log
timeout 900 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo "bench exit $?"
tail -c 600 gpurun_out/r2a/bench.json
