set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ll
for c in 3 4 2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ll/launches_cfg$c.csv python bench.py --config $c --steps 1 --warmup 0 --graph 0 --no-e2e --no-cpu-baseline --no-smooth --no-endpoint > gpurun_out/ll/ncu$c.log 2>&1 || true
done
