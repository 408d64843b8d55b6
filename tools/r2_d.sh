# pass D: device generator tests + timing, compute-sanitizer memcheck
set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2d
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_generate.py -m gpu -x -q > $o/pytest_gen.log 2>&1; echo "pytest exit $?" >> $o/pytest_gen.log
tail -15 $o/pytest_gen.log
python - <<'PY' > $o/gen_time.log 2>&1
import time, torch
from paper_1809_06360_b200 import synth
for c in (1, 4):
    cfg = synth.CONFIGS[c]
    out = synth.generate_batch_device(cfg, seed=0)
    torch.cuda.synchronize()
    t = time.time()
    synth.generate_batch_device(cfg, seed=1, out=out)
    torch.cuda.synchronize()
    print(cfg.name, "device generation s:", time.time() - t, "GB:", sum(v.numel() for v in out.values()) * 8 / 1e9)
    del out
PY
cat $o/gen_time.log
bash tools/sanitize.sh memcheck
