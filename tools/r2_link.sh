# A/B of the link solve: parity (whole GPU suite minus the slow full-size file unless FULL=1), bench lines of configs $@ with and without PLQ_LINK_FUSE
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2link
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $o/pytest.log
for c in ${@:-2 0}; do
 for f in 1 0; do
  PLQ_LINK_FUSE=$f timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-smooth --no-endpoint > $o/bench_cfg${c}_fuse$f.json 2> $o/bench_cfg${c}_fuse$f.err
  python -c "import json; d=json.loads(open('$o/bench_cfg${c}_fuse$f.json').read().strip().splitlines()[-1]); print('cfg$c fuse$f', d['value'], d['ms_per_step'], d.get('phases_ms'), d.get('gpu_launches'), d.get('parity_checked',{}).get('pass'))"
 done
done
