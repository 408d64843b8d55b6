"""Turn a refresh run (gpurun_out/refresh) into the judged evidence under
profiles/<round>/refresh: bench / reference JSON lines, ncu launch-list
summaries, and for every full capture its details CSV, raw-metric summary and
per-source-line stall attribution.

    python tools/process_refresh.py gpurun_out/refresh profiles/r01/refresh
"""
import csv
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def launch_summary(path, title):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rd = csv.reader(lines)
    h = next(rd)
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = {}
    for r in rd:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    # values are in the unit ncu chose (ns or us); report shares, totals in the CSV's unit
    tot = sum(t for _, t in agg.values()) or 1.0
    out = [title, "kernel | launches | total (ncu unit) | share"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{name} | {n} | {t:.1f} | {100 * t / tot:.1f}%")
    return "\n".join(out) + "\n"


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    for f in glob.glob(os.path.join(src, "*.json")):
        shutil.copy(f, dst)
    for f in glob.glob(os.path.join(src, "launches_*.csv")) + glob.glob(os.path.join(src, "sweep_traffic_*.csv")):
        shutil.copy(f, dst)
    for f in glob.glob(os.path.join(src, "launches_*.csv")):
        base = os.path.basename(f)[:-4]
        with open(os.path.join(dst, base + "_summary.txt"), "w") as fh:
            fh.write(launch_summary(f, f"ncu launch list {base} (--metrics gpu__time_duration.sum --clock-control none)"))
    for rep in glob.glob(os.path.join(src, "*.ncu-rep")):
        base = os.path.basename(rep)[:-8]
        if not base.endswith("_full"):
            base += "_full"
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(dst, base + "_details.csv"), "w") as fh:
            fh.write(det)
        summ = subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), rep], capture_output=True,
                              text=True).stdout
        kern = summ.splitlines()[0][3:].split("(")[0].split("::")[-1].split("<")[0] if summ else "."
        src_lines = subprocess.run([sys.executable, os.path.join(HERE, "src_lines.py"), rep, kern, "30"],
                                   capture_output=True, text=True).stdout
        with open(os.path.join(dst, base + "_summary.txt"), "w") as fh:
            fh.write(summ + "\n-- per source line (instructions %, stall samples %) --\n" + src_lines)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
