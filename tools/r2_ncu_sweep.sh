# ncu --set full of the specialized sweep kernels (cfg4 one wave, cfg1 full)
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
python tools/run_sweep.py --config 4 --B 148 --reps 2 > gpurun_out/ncu/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o gpurun_out/ncu/cfg4_sweep python tools/run_sweep.py --config 4 --B 148 --reps 2 > gpurun_out/ncu/ncu4.log 2>&1
echo "ncu4 $?"
python tools/run_sweep.py --config 1 --reps 2 > gpurun_out/ncu/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o gpurun_out/ncu/cfg1_sweep python tools/run_sweep.py --config 1 --reps 2 > gpurun_out/ncu/ncu1.log 2>&1
echo "ncu1 $?"
