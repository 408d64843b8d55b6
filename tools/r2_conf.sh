# shared-memory bank-conflict attribution per source line of the cfg1 / cfg2 sweeps
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2conf
mkdir -p $o
for c in 1 2; do
  B=""; [ $c = 1 ] && B="--B 1024"
  python tools/run_sweep.py --config $c $B --reps 2 > $o/plain$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_small_kernel -s 1 -c 1 -o $o/cfg${c}_sweep python tools/run_sweep.py --config $c $B --reps 2 > $o/ncu$c.log 2>&1
  echo "ncu$c $?"
  python tools/src_conflicts.py $o/cfg${c}_sweep.ncu-rep sweep_small_kernel 45 > $o/conflicts_cfg$c.txt 2>&1
  python tools/src_lines.py $o/cfg${c}_sweep.ncu-rep sweep_small_kernel 45 > $o/stalls_cfg$c.txt 2>&1
done
rm -f $o/*.ncu-rep
head -50 $o/conflicts_cfg1.txt
