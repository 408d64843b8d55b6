# Round-end evidence refresh (run on the GPU box via gpurun).
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/refresh
for c in 1 0 2 3 4; do
  timeout 900 python bench.py --config $c > gpurun_out/refresh/bench_cfg$c.json 2> gpurun_out/refresh/bench_cfg$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/refresh/reference_arm_default.json 2> gpurun_out/refresh/reference_arm_default.err
timeout 300 python bench.py > gpurun_out/refresh/bench_default.json 2> gpurun_out/refresh/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/refresh/launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_launch.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep_small_kernel -c 1 --csv --log-file gpurun_out/refresh/sweep_traffic_cfg1.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_traffic.log 2>&1
ls gpurun_out/refresh
# full ncu captures of the three cfg1 kernels (one launch each)
for k in sweep_small_kernel link_seq_kernel recon_seg_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/refresh/cfg1_$k -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_full_$k.log 2>&1 || true
done
# full ncu captures of the dominant (sweep) kernel of the large-n configs, one launch each
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -c 1 -o gpurun_out/refresh/cfg4_sweep_small_kernel_full -f python bench.py --config 4 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_full_cfg4.log 2>&1 || true
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/refresh/cfg3_sweep_kernel_full -f python bench.py --config 3 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_full_cfg3.log 2>&1 || true
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/refresh/launches_cfg4.csv python bench.py --config 4 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_launch4.log 2>&1 || true
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/refresh/launches_cfg3.csv python bench.py --config 3 --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/refresh/ncu_launch3.log 2>&1 || true
ls gpurun_out/refresh
