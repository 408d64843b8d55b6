# quick A/B loop: parity tests of the sweeps, then the device-resident bench line of the configs given ($@, default 1 2 4)
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2ab
mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > $o/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $o/pytest.log
for c in ${@:-1 2 4}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
  python -c "import json; d=json.loads(open('$o/bench_cfg$c.json').read().strip().splitlines()[-1]); print('cfg$c', d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
done
