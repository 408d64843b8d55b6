set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/exp
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/exp/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/exp/pytest.log
tail -2 gpurun_out/exp/pytest.log
for c in 4 2; do for fz in 0 1; do
  PLQ_RECON_FUSED=$fz timeout 600 python bench.py --config $c --no-cpu-baseline --no-smooth --no-endpoint --no-e2e > gpurun_out/exp/r${c}_$fz.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/exp/r${c}_$fz.json').read().strip().splitlines()[-1]); print('cfg$c fused=$fz', d['value'], d['ms_per_step'], d['phases_ms'])"
done; done
