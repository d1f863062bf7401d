"""Per-stage instruction profile of a barrier-phased kernel in an ncu report:
the SASS is cut at every BAR instruction and each segment's executed
instructions, shared-memory wavefronts (and excess), stall samples and top
opcodes are printed.  For subtree_reg_kernel the three large segments are
stage A (level q0 -> q0+1 into shared memory), stage B (register subtree:
expansion, leaves, contraction) and stage C (level q0+1 -> q0 to HBM).
    python tools/sass_stages.py <rep> [min_instructions]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    floor = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, data = rows[1], rows[2:]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    iW, iX = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")
    iSm = h.index("Warp Stall Sampling (All Samples)")
    segs, cur = [], None

    def fresh(k):
        return {"start": k, "n": 0, "wf": 0, "xs": 0, "samp": 0, "ops": {}}

    cur = fresh(0)
    for k, r in enumerate(data):
        src = r[iS].strip().split()
        if not src:
            continue
        op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
        ex = int(r[iE] or 0)
        cur["n"] += ex
        cur["wf"] += int(r[iW] or 0)
        cur["xs"] += int(r[iX] or 0)
        cur["samp"] += int(r[iSm] or 0)
        cur["ops"][op] = cur["ops"].get(op, 0) + ex
        if op == "BAR":
            cur["end"] = k
            segs.append(cur)
            cur = fresh(k + 1)
    cur["end"] = len(data) - 1
    segs.append(cur)
    tot_s = sum(s["samp"] for s in segs) or 1
    tot_n = sum(s["n"] for s in segs) or 1
    for s in segs:
        if s["n"] < floor:
            continue
        top = sorted(s["ops"].items(), key=lambda x: -x[1])[:9]
        print(f"SASS {s['start']}-{s['end']}: {s['n'] / 1e6:.1f}M inst ({100 * s['n'] / tot_n:.1f}%), "
              f"stall samples {100 * s['samp'] / tot_s:.1f}%, shared wavefronts {s['wf'] / 1e6:.1f}M "
              f"(excess {s['xs'] / 1e6:.1f}M)")
        print("   " + " ".join(f"{o} {c / 1e6:.1f}M" for o, c in top))


if __name__ == "__main__":
    main()
