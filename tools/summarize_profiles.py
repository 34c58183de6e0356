#!/usr/bin/env python3
"""Summarise a profiling pass (tools/profile_all.sh + the bench launch list) into profiles/.

    python tools/summarize_profiles.py <tag> [bench_json]
Writes profiles/<tag>_summary.md, profiles/<tag>_launch_shares.csv and updates
profiles/traffic.json (DRAM bytes per launch of each kernel's full capture).
"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("gps::", "")}
        for w in WANT:
            if w in h:
                d[w] = (r[h.index(w)], units[h.index(w)])
        res.append(d)
    return res


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    tag = sys.argv[1]
    bench = sys.argv[2] if len(sys.argv) > 2 else None
    os.makedirs(P, exist_ok=True)
    lines = [f"# Profile summary {tag}", ""]
    if bench and os.path.exists(bench):
        d = json.load(open(bench))
        lines += [f"Bench line (`{os.path.basename(bench)}`): value **{d['value']} {d['unit']}**, "
                  f"{d['ms_per_step']} ms/step (10 frames), e2e {(d.get('e2e') or {}).get('value')} frames/s, "
                  f"gpu_launches {d['gpu_launches']}, clocks {d['clocks']}", "",
                  f"Roofline: `{json.dumps(d['roofline'])}`", "",
                  "Live CUDA-event shares of the timed region (bench):", "",
                  "| kernel | ms/step | launches/step | share |", "|---|---|---|---|"]
        for k, v in sorted(d["kernels"].items(), key=lambda x: -x[1]["ms_per_step"]):
            lines.append(f"| {k} | {v['ms_per_step']} | {v['launches_per_step']} | {v['share']} |")
        lines.append("")
    lf = os.path.join(G, f"launches_{tag}.csv")
    if os.path.exists(lf):
        rows = [r for r in csv.reader(open(lf)) if len(r) > 10]
        h = rows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for r in rows[1:]:
            name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("gps::", "")
            v = float(r[vi].replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
            tot[name] += v
            cnt[name] += 1
        T = sum(tot.values())
        with open(os.path.join(P, f"{tag}_launch_shares.csv"), "w") as f:
            f.write("kernel,launches,total_ms,share,avg_us\n")
            for k, v in sorted(tot.items(), key=lambda x: -x[1]):
                f.write(f"{k},{cnt[k]},{v / 1e6:.3f},{v / T:.4f},{v / cnt[k] / 1e3:.1f}\n")
        lines += [f"ncu launch list of the same bench command (`ncu --metrics gpu__time_duration.sum "
                  f"--clock-control none`, cold-cache and serialised; compare shares): "
                  f"`profiles/{tag}_launch_shares.csv`", "",
                  "| kernel | launches | share | avg us |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
            lines.append(f"| {k} | {cnt[k]} | {v / T:.3f} | {v / cnt[k] / 1e3:.1f} |")
        lines.append("")
    traffic_path = os.path.join(P, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    lines += ["Full captures (`ncu --set full`, one launch each, tools/profile_all.sh on the steady cfg4 state "
              "of tools/kernel_bench.py):", "",
              "| kernel | us | DRAM read MB | DRAM write MB | warp-inst M | warps active % | regs | lanes/inst | "
              "L2 hit % | L1 hit % | issue active % |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for rep in sorted(glob.glob(os.path.join(G, f"full_{tag}_*.ncu-rep"))):
        for d in raw(rep):
            g = lambda k: d.get(k, ("-", ""))[0]
            rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else 0
            wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else 0
            dur = float(g("gpu__time_duration.sum").replace(",", ""))
            dur_us = dur / 1e3 if d["gpu__time_duration.sum"][1] in ("ns", "nsecond") else dur * (1e3 if d["gpu__time_duration.sum"][1] == "msecond" else 1)
            traffic[d["kernel"].split("<")[0]] = int(rd + wr)
            lines.append(f"| {d['kernel'][:28]} | {dur_us:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                         f"{float(g('smsp__inst_executed.sum')) / 1e6:.1f} | {g('sm__warps_active.avg.pct_of_peak_sustained_active')[:5]} | "
                         f"{g('launch__registers_per_thread')} | {g('smsp__thread_inst_executed_per_inst_executed.ratio')[:5]} | "
                         f"{g('lts__t_sector_hit_rate.pct')[:5]} | {g('l1tex__t_sector_hit_rate.pct')[:5]} | "
                         f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active')[:5]} |")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
