#!/usr/bin/env python3
"""Hot spots of an ncu report (captured with -lineinfo and --import-source on): CUDA source lines
ranked by warp-stall samples, with their share of executed instructions.
    python tools/ncu_hot.py <report.ncu-rep> [n]"""
import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    stall = collections.Counter()
    inst = collections.Counter()
    text = {}
    f = "?"
    cols = None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            cols = r
            continue
        if cols is None or r[0] in ("Function Name",):
            continue
        try:
            ln = int(r[0])
            s = int(r[4] or 0)
            i = int(r[7] or 0)
        except (ValueError, IndexError):
            continue
        key = (f, ln)
        stall[key] += s
        inst[key] += i
        if r[1].strip():
            text[key] = r[1].strip()[:100]
    ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
    print(f"total stall samples {ts}, warp instructions {ti}")
    for key, s in stall.most_common(n):
        print(f"{100 * s / ts:5.1f}% stall {100 * inst[key] / ti:5.1f}% inst  {key[0]}:{key[1]:<5} {text.get(key, '')}")


if __name__ == "__main__":
    main()
