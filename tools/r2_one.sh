# refresh one config's evidence (bench line, reference arm, ncu launch list): bash tools/r2_one.sh 2
set -u
cd $GRAFT_REPO_ROOT
c=$1
o=gpurun_out/r2one
mkdir -p $o
timeout 900 python bench.py --config $c > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
timeout 600 python bench.py --config $c --impl reference > $o/reference_cfg$c.json 2> $o/reference_cfg$c.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg$c.csv \
  python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint --no-parity > $o/ncu_launch_cfg$c.log 2>&1
python tools/process_refresh.py $o $o/processed > $o/process.log 2>&1
python -c "import json; d=json.loads(open('$o/bench_cfg$c.json').read().strip().splitlines()[-1]); print('cfg$c', d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('e2e',{}).get('value'), d.get('parity_checked',{}).get('pass'))"
ls $o/processed
