# pass C: new tests (multi-rank native sharded entry through the host shim, chain link solve), default bench
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2c
mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -m gpu -x -q -k "multi_rank or chain_link" > $o/pytest_new.log 2>&1; echo "pytest exit $?" >> $o/pytest_new.log
tail -30 $o/pytest_new.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_default.json 2> $o/bench_default.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$o/bench_default.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
python tools/run_sweep.py --config 3 --reps 2 > $o/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o $o/cfg3_sweep python tools/run_sweep.py --config 3 --reps 2 > $o/ncu3.log 2>&1
echo "ncu3 $?"
