set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2q4
mkdir -p $o
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg4.json 2> $o/bench_cfg4.err
python -c "import json; d=json.loads(open('$o/bench_cfg4.json').read().strip().splitlines()[-1]); print(4, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
timeout 900 python bench.py --config 2 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg2.json 2> $o/bench_cfg2.err
python -c "import json; d=json.loads(open('$o/bench_cfg2.json').read().strip().splitlines()[-1]); print(2, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
PLQ_LIB_PATH=$GRAFT_REPO_ROOT/paper_1809_06360_b200/libparlqr_b200_prof.so python tools/phase_profile.py --config 4 --B 148 > $o/phase_cfg4.json 2>&1
python -c "import json; d=json.load(open('$o/phase_cfg4.json')); print(d['sweep_ms']); [print(f'{v:10.0f}  {k}') for k,v in d['cycles_per_stage_by_phase'].items()]"
