# phase profile (measurement build), failing / new tests, cfg1 launch list
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
bash tools/r2_phase.sh > gpurun_out/r2c/phase.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -s -rf -k "full_size or host_entry" > gpurun_out/r2c/t.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2c/t.log
tail -3 gpurun_out/r2c/t.log
python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e --no-parity > gpurun_out/r2c/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_cfg1.csv python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e --no-parity > gpurun_out/r2c/ncu.log 2>&1
echo "ncu exit $?"
