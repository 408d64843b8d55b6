# round-2 final evidence: GPU suite, smoke, bench lines + reference arms of every config, launch lists, full
# ncu captures of every config's sweep kernel (processed into profiles/r02/final by tools/process_refresh.py)
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2final
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -3 $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke exit $?" >> $o/smoke.log
tail -2 $o/smoke.log
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference > $o/reference_default.json 2> $o/reference_default.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_default.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint --no-parity > $o/ncu_launch_default.log 2>&1
for c in 0 1 2 3; do
  timeout 900 python bench.py --config $c > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
  timeout 600 python bench.py --config $c --impl reference > $o/reference_cfg$c.json 2> $o/reference_cfg$c.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint --no-parity > $o/ncu_launch_cfg$c.log 2>&1
done
for c in default cfg0 cfg1 cfg2 cfg3; do
  python -c "import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('e2e',{}).get('value'), d.get('parity_checked',{}).get('pass'))"
done
python tools/run_sweep.py --config 4 --B 148 --reps 2 > $o/plain4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o $o/cfg4_sweep python tools/run_sweep.py --config 4 --B 148 --reps 2 > $o/ncu4.log 2>&1
echo "ncu4 $?"
for c in 1 2; do
python tools/run_sweep.py --config $c --reps 2 > $o/plain$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o $o/cfg${c}_sweep python tools/run_sweep.py --config $c --reps 2 > $o/ncu$c.log 2>&1
echo "ncu$c $?"
done
python tools/run_sweep.py --config 3 --reps 2 > $o/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o $o/cfg3_sweep python tools/run_sweep.py --config 3 --reps 2 > $o/ncu3.log 2>&1
echo "ncu3 $?"
# summaries on the box (details CSV, raw-metric summary, per-source-line stalls); the .ncu-rep files stay there
# (gpurun_out is capped at 64 MiB)
python tools/process_refresh.py $o $o/processed > $o/process.log 2>&1
rm -f $o/*.ncu-rep
du -sh $o
