"""Algorithmic work counts of the partitioned solve, used for
roofline fractions.  Flops are the reference's own formulas with each
distinct product counted once; bytes are the compulsory inputs plus outputs.

Per endpoint stage  F_e = 6n^3 + 20n^2 m + 12 n m^2 + m^3/3 + 20n^2 + 16nm + 7m^2
Per serial stage    F_s = 4n^3 + 8n^2 m + 8 n m^2 + m^3/3 + 11n^2 + 9nm + 5m^2
Per knot (recon)    F_r = 14n^2 + 18nm + 4m^2
Per link block      F_l = 13n^3/3 + 6n^2
"""

from __future__ import annotations

import json
import os

FP64_PEAK_FILE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                              "profiles", "fp64_peak.json")
# Measured on this pool's B200 by tools/fp64_peak.cu (DFMA and DMMA.8x8x4
# both at 37.0 TFLOP/s, 148 SMs at 1965 MHz): the FP64 roofline denominator
# MEASURED_PEAKS.json does not carry.
FP64_PEAK_TFLOPS_DEFAULT = 37.0


def fp64_peak_tflops():
    try:
        with open(FP64_PEAK_FILE) as fh:
            d = json.load(fh)
        vals = [v for k, v in d.items() if k.endswith("_tflops")]
        return max(vals) if vals else FP64_PEAK_TFLOPS_DEFAULT
    except (OSError, ValueError):
        return FP64_PEAK_TFLOPS_DEFAULT


def hbm_peak_gbs(repo_root=None):
    root = repo_root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


def sweep_kernel_name(n, m, force_generic=False):
    """The K1 kernel the C-ABI layer picks for (n, m) (plq_api.cu
    use_small_sweep / sweep_threads), named as ncu lists it."""
    small = {(12, 4): "sweep_small_kernel<12,4,1,1>", (32, 8): "sweep_small_kernel<32,8,4,1>",
             (64, 32): "sweep_small_kernel<64,32,8,1>"}
    if not force_generic and (n, m) in small:
        return small[(n, m)]
    nt = 32 if n <= 16 else (128 if n <= 32 else 256)
    return f"sweep_kernel<{nt}>"


def stage_flops(n, m):
    Fe = 6 * n**3 + 20 * n**2 * m + 12 * n * m**2 + m**3 / 3 + 20 * n**2 + 16 * n * m + 7 * m**2
    Fs = 4 * n**3 + 8 * n**2 * m + 8 * n * m**2 + m**3 / 3 + 11 * n**2 + 9 * n * m + 5 * m**2
    Fr = 14 * n**2 + 18 * n * m + 4 * m**2
    Fl = 13 * n**3 / 3 + 6 * n**2
    return Fe, Fs, Fr, Fl


def problem_flops(n, m, T, J):
    """Total algorithmic flops of one problem and of its sweep phase."""
    L = T / J
    Fe, Fs, Fr, Fl = stage_flops(n, m)
    sweep = (J - 1) * L * Fe + L * Fs
    total = sweep + T * Fr + (J - 1) * Fl
    return total, sweep


def knot_bytes(n, m):
    """Compulsory bytes per knot: inputs read once, outputs written once."""
    return 8 * (2 * n * n + 2 * n * m + m * m + 2 * n + m), 8 * (n * m + 2 * m + 2 * n)


def sweep_bytes(n, m, T, J):
    """Compulsory HBM bytes of the sweep kernel for one problem: stage inputs
    read once, K/Kz/k1 written, segment-start value blocks written."""
    bin_, _ = knot_bytes(n, m)
    return T * bin_ + T * 8 * (2 * n * m + m) + J * 8 * (3 * n * n + 2 * n)
