# pass L: cfg4 / cfg2 phase profiles (measurement build), then the whole GPU suite
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2l
mkdir -p $o
PLQ_LIB_PATH=$GRAFT_REPO_ROOT/paper_1809_06360_b200/libparlqr_b200_prof.so python tools/phase_profile.py --config 4 --B 148 > $o/phase_cfg4.json 2>&1
python -c "import json; d=json.load(open('$o/phase_cfg4.json')); print(d['sweep_ms']); [print(f'{v:10.0f}  {k}') for k,v in d['cycles_per_stage_by_phase'].items()]"
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -4 $o/pytest.log
