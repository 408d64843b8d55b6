# A/B of the forward solve fused into the link elimination's factorization (PLQ_LINK_FSOLVE)
set -u
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
for c in 2; do for f in 1 0 1 0; do
  PLQ_LINK_FSOLVE=$f python bench.py --config $c --no-cpu-baseline --no-e2e --no-smooth --no-endpoint 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$c fsolve$f', d['ms_per_step'], d['phases_ms'], d['gpu_launches'], d['parity_checked']['pass'])"
done; done
