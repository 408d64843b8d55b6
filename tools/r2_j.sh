# per-phase cycles of the generic sweep on cfg3 (measurement build)
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2j2
mkdir -p $o
PLQ_LIB_PATH=$GRAFT_REPO_ROOT/paper_1809_06360_b200/libparlqr_b200_prof.so python tools/phase_profile.py --generic --config 3 > $o/phase_cfg3.json 2>&1
cat $o/phase_cfg3.json
