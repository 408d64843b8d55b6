set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/large
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/large/cfg3_sweep_full -f python bench.py --config 3 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/large/ncu3f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:link_backsub -c 2 -o gpurun_out/large/cfg3_backsub -f python bench.py --config 3 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/large/ncu3b.log 2>&1
