set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/exp
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/exp/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/exp/pytest.log
tail -2 gpurun_out/exp/pytest.log
for th in 256 512; do
  PLQ_SWEEP_THREADS=$th timeout 600 python bench.py --config 3 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e > gpurun_out/exp/b3_$th.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/exp/b3_$th.json').read().strip().splitlines()[-1]); print('cfg3 threads $th', d['value'], d['ms_per_step'], d['phases_ms'], round(d['roofline']['frac'],4))"
done
