# after the lane-parallel stage copies: phase profile, parity tests, quick bench of all configs
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2e
bash tools/r2_phase.sh > gpurun_out/r2e/phase.log 2>&1
cp gpurun_out/phase/*.json gpurun_out/r2e/
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_endpoint.py tests/test_gpu_smooth.py -m gpu -q -x > gpurun_out/r2e/t.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2e/t.log
tail -2 gpurun_out/r2e/t.log
for c in 1 2 3 4; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e --no-parity > gpurun_out/r2e/bench_cfg$c.json 2>gpurun_out/r2e/bench_cfg$c.err
python -c "import json; d=json.loads(open('gpurun_out/r2e/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['phases_ms'], round(d['roofline']['frac'],4))"
done
