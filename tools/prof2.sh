set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -c 1 -o gpurun_out/p2/cfg2_sweep -f python bench.py --config 2 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/p2/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recon_kernel -c 1 -o gpurun_out/p2/cfg3_recon -f python bench.py --config 3 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/p2/ncu3r.log 2>&1
