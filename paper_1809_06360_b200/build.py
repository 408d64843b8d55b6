"""Build the sm_100a CUDA library ``libparlqr_b200.so`` in-tree.

``python -m paper_1809_06360_b200.build`` (also called by
``__graft_entry__.build()``).  Plain nvcc, no torch extension machinery: the
product is a C-ABI shared library (include/parlqr_b200.h) loaded by ctypes.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libparlqr_b200.so")
SOURCES = ("plq_sweep.cu", "plq_sweep_t32.cu", "plq_sweep_t128.cu", "plq_sweep_t256.cu", "plq_sweep_t512.cu", "plq_sweep_small.cu", "plq_link.cu", "plq_recon.cu", "plq_recon_small.cu", "plq_recon_ring.cu",
           "plq_smooth.cu", "plq_endpoint.cu", "plq_linkfeas.cu", "plq_linkchain.cu", "plq_generate.cu",
           "plq_api.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "parlqr_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, profile=False):
    """``profile=True``: a measurement build with the sweep's per-phase cycle
    counters (-DPLQ_PHASE_PROFILE) as libparlqr_b200_prof.so (load it with
    PLQ_LIB_PATH); the product library never has them."""
    lib_path = LIB.replace(".so", "_prof.so") if profile else LIB
    if not force and not profile and not _stale():
        return LIB
    objdir = os.path.join(HERE, "_build_prof" if profile else "_build")
    flags = FLAGS + (["-DPLQ_PHASE_PROFILE"] if profile else [])
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, src.replace(".cu", ".o")) for src in SOURCES]
    # translation units are independent: compile them concurrently
    # (objects newer than their source and every header are kept unless forced)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")]
    hdrs.append(os.path.join(ROOT, "include", "parlqr_b200.h"))
    hdr_t = max(os.path.getmtime(h) for h in hdrs)
    todo = [(src, obj) for src, obj in zip(SOURCES, objs)
            if force or not os.path.exists(obj)
            or os.path.getmtime(obj) <= max(hdr_t, os.path.getmtime(os.path.join(CSRC, src)))]
    procs = [subprocess.Popen([nvcc(), *ARCH, *flags, "-c", os.path.join(CSRC, src), "-o", obj],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for src, obj in todo]
    log = []
    failed = []
    for (src, _), p in zip(todo, procs):
        out, _ = p.communicate()
        log.append(out)
        if p.returncode:
            failed.append(f"nvcc failed for {src}:\n{out}")
    if failed:
        raise RuntimeError("\n".join(failed))
    tmp = lib_path + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib_path)
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
