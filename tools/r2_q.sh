# quick loop: cfg3 bench line (+ generic phase profile when the measurement build is present) and the large-n tests
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2q
mkdir -p $o
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg3.json 2> $o/bench_cfg3.err
python -c "import json; d=json.loads(open('$o/bench_cfg3.json').read().strip().splitlines()[-1]); print(3, d['value'], d['ms_per_step'], d.get('phases_ms'), round(d['roofline']['frac'],4), d.get('parity_checked',{}).get('pass'))"
if [ -f paper_1809_06360_b200/libparlqr_b200_prof.so ]; then
PLQ_LIB_PATH=$GRAFT_REPO_ROOT/paper_1809_06360_b200/libparlqr_b200_prof.so python tools/phase_profile.py --generic --config 3 > $o/phase_cfg3.json 2>&1
python -c "import json; d=json.load(open('$o/phase_cfg3.json')); print(d['sweep_ms']); [print(f'{v:10.0f}  {k}') for k,v in d['cycles_per_stage_by_phase'].items()]"
fi
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -m gpu -x -q -k "split or cfg3 or big or n128 or 128 or multi_rank" 2>&1 | tail -3
