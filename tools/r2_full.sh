# round-2 evidence pass: full GPU suite, smoke, default bench (cfg4), other configs, launch list of the default bench
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2f
mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -3 $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke exit $?" >> $o/smoke.log
tail -2 $o/smoke.log
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench exit $?"
tail -c 3000 $o/bench_default.json
for c in 1 2 3; do
  timeout 900 python bench.py --config $c > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
  python -c "import json; d=json.loads(open('$o/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('e2e',{}).get('value'))"
done
