# pass G: cfg3 bench after storing Mzu' straight into P, generic-path tests
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2i
mkdir -p $o
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python -c "import json; d=json.loads(open('$o/bench_cfg3.json').read().strip().splitlines()[-1]); print(3, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -3 $o/pytest.log
