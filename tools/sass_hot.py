#!/usr/bin/env python3
"""Per-SASS-instruction hot spots of one ncu capture (source page, sass view).

    python tools/sass_hot.py <report.ncu-rep> [top] [--range A B]
Prints the instructions with the most warp-stall samples and the most executed warp
instructions, plus totals, so a kernel's time can be attributed to its loop body."""
import csv
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        data.append(d)
    return h, data


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 30
    h, data = load(rep)
    stall_cols = [c for c in h if c.startswith("stall_")]
    tot_s = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
    tot_i = sum(num(d["Instructions Executed"]) for d in data)
    print(f"samples {tot_s:.0f}  warp-instr {tot_i:.0f}  instructions {len(data)}")
    agg = {c: sum(num(d[c]) for d in data) for c in stall_cols}
    print("stall reasons:", ", ".join(f"{c[6:]}={v / tot_s:.2f}" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for i, d in enumerate(data):
        d["_i"] = i
    hot = sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:top]
    for d in sorted(hot, key=lambda d: d["_i"]):
        s = num(d["Warp Stall Sampling (All Samples)"])
        main_stall = max(stall_cols, key=lambda c: num(d[c]))
        print(f"{d['_i']:5d} {d['Address'][-5:]} {s / tot_s * 100:5.1f}% ex={num(d['Instructions Executed']) / 1e6:6.2f}M "
              f"thr={num(d['Avg. Threads Executed']):4.1f} {main_stall[6:]:>16s}  {d['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
