# round 2 GPU check: whole GPU suite (incl. full-size, cross-term, rank-repair, 2-rank) + quick bench of cfg1-3
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 2400 python -m pytest tests -m gpu -q -s -rA --durations=25 > gpurun_out/r2b/t_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2b/t_all.log
grep -E "passed|failed|error" gpurun_out/r2b/t_all.log | tail -5
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-smooth --no-endpoint --no-e2e > gpurun_out/r2b/bench_cfg$c.json 2> gpurun_out/r2b/bench_cfg$c.err
  python -c "import json; d=json.loads(open('gpurun_out/r2b/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['phases_ms'], round(d['roofline']['frac'],4), d['parity_checked']['pass_K_objective_1e-9'])"
done
