"""Render the DESIGN.md results table from bench JSON lines.

    python tools/results_table.py profiles/r01/refresh

reads bench_cfg{0..4}.json (+ reference_arm_*.json if present) and prints
a markdown table: device-resident knots/s, ms/step, phases, sweep FP64
fraction, e2e knots/s (+ copy-roofline fraction), smoothing and endpoint legs,
CPU baselines.
"""

import json
import os
import sys


def last_json(path):
    with open(path) as fh:
        lines = [ln for ln in fh.read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def fmt(v, unit=""):
    if v is None:
        return "—"
    if abs(v) >= 1e6:
        return f"{v / 1e6:.3g}M{unit}"
    if abs(v) >= 1e3:
        return f"{v / 1e3:.3g}k{unit}"
    return f"{v:.3g}{unit}"


def main(d):
    rows = []
    for c in range(5):
        p = os.path.join(d, f"bench_cfg{c}.json")
        if not os.path.exists(p):
            continue
        j = last_json(p)
        if not j:
            continue
        ph = j.get("phases_ms", {})
        e2e = j.get("e2e") or {}
        cr = e2e.get("copy_roofline") or {}
        sm = j.get("smooth") or {}
        ep = j.get("endpoint") or {}
        cpu = j.get("cpu_baseline") or {}
        rows.append("| {} | {} | {:.3f} | {:.3f} / {:.3f} / {:.3f} | {:.3f} | {} ({}) | {} | {} | {} ({} cores) |".format(
            c, fmt(j["value"]), j["ms_per_step"], ph.get("sweep", 0), ph.get("link", 0), ph.get("recon", 0),
            j["roofline"]["frac"], fmt(e2e.get("value")), f"{cr['frac']:.2f} of PCIe" if cr else "—",
            f"{fmt(sm.get('value'))} / {sm['ms_per_step']:.3g} ms" if sm else "—",
            f"{fmt(ep.get('value'))} / {ep['ms_per_step']:.3g} ms" if ep else "—",
            fmt(cpu.get("value")), cpu.get("cores", "—")))
    print("| cfg | knots/s (device) | ms/step | sweep / link / recon ms | sweep FP64 frac | e2e knots/s | "
          "smooth knots/s / ms | endpoint knots/s / ms | CPU port knots/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(r)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01/refresh")
