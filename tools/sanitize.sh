# compute-sanitizer evidence: ONE tool per call (tools/sanitize.sh memcheck|racecheck|synccheck|initcheck)
# over the solve of small instances of every kernel family (specialized n = 12 / 32 / 64, generic n = 128,
# generic odd shapes incl. the rank-repair pass)
set -u
cd $GRAFT_REPO_ROOT
tool=$1
mkdir -p gpurun_out/sanitize
out=gpurun_out/sanitize/$tool.log
: > $out
run() {
  echo "== $*" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 "$@" >> $out 2>&1
  echo "exit $?" >> $out
}
run python tools/run_sweep.py --config 1 --B 32 --phase solve --reps 1
run python tools/run_sweep.py --config 2 --T 512 --J 8 --phase solve --reps 1
run python tools/run_sweep.py --config 4 --B 2 --T 128 --J 4 --phase solve --reps 1
run python tools/run_sweep.py --config 3 --T 64 --J 4 --phase solve --reps 1
run python tools/rank_case.py
grep -E "^== |^exit|ERROR SUMMARY" $out
