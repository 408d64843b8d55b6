# re-entry check: GPU suite, smoke, default bench line (one gpurun call)
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2check
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -3 $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke exit $?" >> $o/smoke.log
tail -2 $o/smoke.log
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench exit $?"
tail -c 3000 $o/bench_default.json
