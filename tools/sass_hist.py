"""Opcode histogram (+stall share, excess smem wavefronts) of one kernel in an ncu report.
    python tools/sass_hist.py <rep> [top]"""
import csv
import subprocess
import sys
from collections import Counter


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    data = rows[2:]
    ie, ss = idx["Instructions Executed"], idx["Warp Stall Sampling (All Samples)"]
    ex = idx.get("L1 Wavefronts Shared Excessive")
    tot = sum(int(r[ie] or 0) for r in data)
    samp = sum(int(r[ss] or 0) for r in data) or 1
    c, s, x = Counter(), Counter(), Counter()
    for r in data:
        parts = r[idx["Source"]].split()
        if not parts:
            continue
        op = parts[1] if parts[0].startswith("@") else parts[0]
        op = op.split(".")[0]
        c[op] += int(r[ie] or 0)
        s[op] += int(r[ss] or 0)
        x[op] += int(r[ex] or 0) if ex is not None else 0
    print(f"total warp instructions {tot / 1e6:.1f}M")
    for op, v in c.most_common(top):
        print(f"{op:10s} {v / 1e6:9.1f}M {100 * v / tot:5.1f}%  stall {100 * s[op] / samp:5.1f}%  excess_wf {x[op] / 1e6:.1f}M")


if __name__ == "__main__":
    main()
