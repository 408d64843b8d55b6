set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/exp
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/exp/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/exp/pytest.log
tail -2 gpurun_out/exp/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/exp/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/exp/smoke.log; tail -2 gpurun_out/exp/smoke.log
for v in 0 1 2; do
  PLQ_RECON_RS=$v timeout 600 python bench.py --config 2 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e > gpurun_out/exp/rs2_$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/exp/rs2_$v.json').read().strip().splitlines()[-1]); print('cfg2 rs=$v', d['ms_per_step'], d['phases_ms'])"
done
