# ncu full captures of the large-n sweep kernels on reduced shapes (run via gpurun)
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/large
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -c 1 -o gpurun_out/large/cfg4_sweep -f python tools/prof_run.py 4 16 1024 32 1 > gpurun_out/large/ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/large/cfg3_sweep -f python tools/prof_run.py 3 1 512 32 1 > gpurun_out/large/ncu3.log 2>&1
