# round-2 evidence pass B: new tests, bench lines of cfg1-3 (+ reference arms), launch lists, ncu --set full of every config's sweep kernel
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2b
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -m gpu -x -q -k "native or unsym" > $o/pytest_new.log 2>&1; echo "pytest exit $?" >> $o/pytest_new.log
tail -15 $o/pytest_new.log
for c in 1 2 3; do
  timeout 900 python bench.py --config $c > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
  python -c "import json; d=json.loads(open('$o/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('e2e',{}).get('value'))"
  timeout 600 python bench.py --config $c --impl reference > $o/reference_cfg$c.json 2> $o/reference_cfg$c.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint --no-parity > $o/ncu_launch_cfg$c.log 2>&1
done
# full captures of the sweep kernels (second sweep launch of run_sweep.py)
python tools/run_sweep.py --config 4 --B 148 --reps 2 > $o/plain4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o $o/cfg4_sweep python tools/run_sweep.py --config 4 --B 148 --reps 2 > $o/ncu4.log 2>&1
echo "ncu4 $?"
for c in 1 2; do
python tools/run_sweep.py --config $c --reps 2 > $o/plain$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o $o/cfg${c}_sweep python tools/run_sweep.py --config $c --reps 2 > $o/ncu$c.log 2>&1
echo "ncu$c $?"
done
python tools/run_sweep.py --config 3 --reps 2 > $o/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o $o/cfg3_sweep python tools/run_sweep.py --config 3 --reps 2 > $o/ncu3.log 2>&1
echo "ncu3 $?"
ls -la $o
