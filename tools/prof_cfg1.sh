set -e
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/prof_plain.json 2>&1
for k in sweep_small_kernel link_seq_kernel recon_seg_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/cfg1_$k -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/ncu_$k.log 2>&1 || true
done
ls -la gpurun_out/*.ncu-rep
