# pass M: cfg4 / cfg2 bench lines after the conflict-free recon dot products + recon parity tests
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2m
mkdir -p $o
for c in 4 2; do
timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
python -c "import json; d=json.loads(open('$o/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -3 $o/pytest.log
