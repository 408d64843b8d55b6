# quick GPU check: full gpu test suite + selected bench configs (args: configs)
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/chk
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/chk/pytest.log
tail -3 gpurun_out/chk/pytest.log
for c in "$@"; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-smooth --no-endpoint --no-e2e > gpurun_out/chk/bench_cfg$c.json 2> gpurun_out/chk/bench_cfg$c.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/chk/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['phases_ms'], round(d['roofline']['frac'],4))"
done
