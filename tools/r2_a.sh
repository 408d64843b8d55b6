# round-2 evidence pass A: full GPU suite, smoke, default bench (cfg4), its reference arm, launch list of the default bench
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2a
mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -3 $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke exit $?" >> $o/smoke.log
tail -2 $o/smoke.log
timeout 900 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench exit $?"
tail -c 3000 $o/bench_default.json
timeout 600 python bench.py --impl reference > $o/reference_default.json 2> $o/reference_default.err; echo "ref exit $?"
tail -c 1000 $o/reference_default.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_default.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-smooth --no-endpoint --no-parity > $o/ncu_launch.log 2>&1
echo "ncu launch exit $?"
