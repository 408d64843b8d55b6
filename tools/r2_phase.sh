# per-phase cycle breakdown of the specialized sweeps (measurement build)
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/phase
export PLQ_LIB_PATH=$GRAFT_REPO_ROOT/paper_1809_06360_b200/libparlqr_b200_prof.so
python tools/phase_profile.py --config 4 --B 148 > gpurun_out/phase/cfg4.json 2>&1
python tools/phase_profile.py --config 1 > gpurun_out/phase/cfg1.json 2>&1
python tools/phase_profile.py --config 2 > gpurun_out/phase/cfg2.json 2>&1
cat gpurun_out/phase/*.json
