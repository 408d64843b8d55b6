"""Per-CUDA-source-line shared-memory wavefronts (total / excessive = bank-conflict replays) from an ncu
report: python tools/src_conflicts.py REPORT KERNEL_REGEX [top]"""
import csv
import subprocess
import sys


def main(path, kernel, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = {}
    fname = "?"
    i = 0
    tw = te = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            h = r
            cols = [c for c in h if "Shared" in c]
            try:
                wi, xi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")
            except ValueError:
                print("columns with 'Shared':", cols)
                return
            i += 1
            cur = None
            while i < len(rows) and rows[i] and rows[i][0] not in ("File Path", "Line No", "Function Name"):
                rr = rows[i]
                if rr[0]:
                    cur = (fname, int(rr[0]), rr[1].strip()[:100])
                try:
                    w, x = float(rr[wi] or 0), float(rr[xi] or 0)
                except ValueError:
                    w, x = 0, 0
                if cur:
                    a = agg.setdefault(cur, [0.0, 0.0])
                    a[0] += w
                    a[1] += x
                tw += w
                te += x
                i += 1
            continue
        i += 1
    print(f"shared wavefronts {tw:.0f}, excessive {te:.0f} ({te / max(tw, 1) * 100:.1f}%)")
    for (f, ln, src), (w, x) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{x / max(te, 1) * 100:5.1f}%x {w / max(tw, 1) * 100:5.1f}%w  {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
