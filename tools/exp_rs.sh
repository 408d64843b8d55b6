set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/exp
for v in 0 1 2; do
  PLQ_RECON_RS=$v timeout 600 python bench.py --config 4 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e > gpurun_out/exp/rs$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/exp/rs$v.json').read().strip().splitlines()[-1]); print('rs=$v', d['ms_per_step'], d['phases_ms'])"
done
