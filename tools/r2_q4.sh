set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2q4
mkdir -p $o
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg4.json 2> $o/bench_cfg4.err
python -c "import json; d=json.loads(open('$o/bench_cfg4.json').read().strip().splitlines()[-1]); print(4, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "chain" 2>&1 | tail -2
