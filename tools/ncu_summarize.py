#!/usr/bin/env python
"""Summarise the round's ncu captures (gpurun_out/) into profiles/.

Writes profiles/ncu_summary_<round>.md (launch shares + key counters of the
dominant kernel per config) and profiles/ncu_traffic.json (dram bytes per
launch of the dominant kernel, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
SRC = os.path.join(ROOT, "gpurun_out")
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            d[h] = (float(v.replace(",", "")), u)
        except ValueError:
            d[h] = (v, u)
    return d


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        name = r[iN].split("(")[0]
        v = float(r[iV].replace(",", "")) * UNIT_SCALE.get(r[iU], 1e-9)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    return [(k, cnt[k], v, v / s) for k, v in tot.most_common()]


def main():
    lines = [f"# ncu summary, round {RND[1:]}", "",
             "Captured on a B200 with `tools/profile_round.sh` (bench.py --steps 3 --warmup 3, one GPU);",
             "launch lists use `--metrics gpu__time_duration.sum --clock-control none` (cold, serialised:",
             "compare shares, not absolutes); full captures use `--set full --clock-control none --cache-control none`.", ""]
    traffic = {}
    for c in (2, 3, 4, 5, 6, 7, 8, 9):
        w = bench.workload(c)
        lines.append(f"## config {c}: {w['name']}")
        lp = os.path.join(SRC, f"launches_c{c}.csv")
        if os.path.exists(lp):
            lines.append("")
            lines.append("| kernel | launches | total ms | share |")
            lines.append("|---|---|---|---|")
            for k, n, v, sh in launch_shares(lp):
                lines.append(f"| `{k}` | {n} | {v * 1e3:.3f} | {100 * sh:.1f}% |")
        rp = os.path.join(SRC, f"full_c{c}.ncu-rep")
        if os.path.exists(rp):
            d = raw_metrics(rp)
            lines.append("")
            lines.append("Full capture of the dominant kernel (one launch):")
            lines.append("")
            for k in KEYS:
                if k in d:
                    v, u = d[k]
                    lines.append(f"- `{k}` = {v} {u}")
            rb = d.get("dram__bytes_read.sum", (0, "byte"))
            wb = d.get("dram__bytes_write.sum", (0, "byte"))
            tb = rb[0] * UNIT_SCALE.get(rb[1], 1) + wb[0] * UNIT_SCALE.get(wb[1], 1)
            traffic[w["name"]] = tb
            lines.append(f"- dram traffic per launch = {tb / 1e9:.4f} GB")
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_summary_{RND}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
