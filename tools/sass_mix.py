"""Instruction mix / stall attribution of one kernel from an ncu report (SASS page)."""
import collections
import csv
import subprocess
import sys


def main(path, kernel, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    mix = collections.Counter()
    stall = collections.Counter()
    for r in rows[2:]:
        if len(r) <= max(si, wi, ei):
            continue
        op = r[si].split()[0] if r[si].split() else "?"
        if op.startswith("@"):
            op = r[si].split()[1]
        op = op.split(".")[0]
        mix[op] += int(r[ei] or 0)
        stall[op] += float(r[wi] or 0)
    ti, ts = sum(mix.values()) or 1, sum(stall.values()) or 1
    print(f"{'op':12s} {'inst%':>7s} {'stall%':>7s}")
    for op, _ in sorted(stall.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{op:12s} {mix[op] / ti * 100:7.1f} {stall[op] / ts * 100:7.1f}")
    print("total instructions", ti)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
