"""Per-CUDA-source-line instruction / stall attribution from an ncu report
(cuda,sass source view): python tools/src_lines.py REPORT KERNEL_REGEX [top]"""
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
    total_i = total_s = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            h = r
            ei, wi = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
            i += 1
            cur = None
            while i < len(rows) and rows[i] and rows[i][0] not in ("File Path", "Line No", "Function Name"):
                rr = rows[i]
                if rr[0]:
                    cur = (fname, int(rr[0]), rr[1].strip()[:90])
                try:
                    ins, st = int(rr[ei] or 0), float(rr[wi] or 0)
                except ValueError:
                    ins, st = 0, 0
                if cur:
                    a = agg.setdefault(cur, [0, 0.0])
                    a[0] += ins
                    a[1] += st
                total_i += ins
                total_s += st
                i += 1
            continue
        i += 1
    print(f"total instructions {total_i}, stall samples {total_s:.0f}")
    for (f, ln, src), (ins, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{ins / max(total_i, 1) * 100:5.1f}%i {st / max(total_s, 1) * 100:5.1f}%s {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
