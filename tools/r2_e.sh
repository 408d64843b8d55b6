# pass E: memory-hygiene tests, cfg3 bench after the value-update preload, default bench with the device generator
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2e
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_memcheck.py -m gpu -x -q > $o/pytest_mem.log 2>&1; echo "pytest exit $?" >> $o/pytest_mem.log
tail -15 $o/pytest_mem.log
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python -c "import json; d=json.loads(open('$o/bench_cfg3.json').read().strip().splitlines()[-1]); print(3, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
( time timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err ) 2>&1 | grep real
python -c "import json; d=json.loads(open('$o/bench_default.json').read().strip().splitlines()[-1]); print(4, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d['roofline']['traffic'], d.get('parity_checked',{}).get('pass'), d['e2e']['value'], d['data'])"
tail -3 $o/bench_default.err
