#!/usr/bin/env python
"""profiles/ncu_summary_<round>.md from a round directory: per-kernel launch means of the ncu launch lists
(launches_c*.csv), key counters of the full captures given on the command line (tools/ncu_keys.py) and
the committed bench lines (bench_c*.json).

usage: tools/round_summary.py profiles/r02 [label=report.ncu-rep ...] > profiles/ncu_summary_r02.md"""
import collections
import csv
import glob
import json
import os
import re
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
         "msecond": 1e3, "inst": 1}
rnd = sys.argv[1]
reports = [a.split("=", 1) for a in sys.argv[2:]]
print(f"# ncu summary, {os.path.basename(rnd)}\n")
print("Captured under `gpurun` on one B200 (1965 MHz, `--clock-control none`). Launch lists: `launches_c<cfg>.csv`")
print("(`gpu__time_duration.sum`, `dram__bytes_read/write.sum`, `smsp__inst_executed.sum` per launch of")
print("`bench.py --steps 3 --warmup 3 --config c`, serialised and cold-cache under ncu: the kernels' shares of a")
print("step, not their absolute times). Full captures: `--set full --cache-control none --import-source on`.\n")
print("## Per-kernel launch means (ncu launch lists)\n")
print("| config | kernel | launches | mean us | DRAM read MB | DRAM write MB | warp instructions (M) |")
print("|---|---|---|---|---|---|---|")
def cfgnum(p): return int(re.search(r"launches_c(\d+)", p).group(1))
for p in sorted(glob.glob(os.path.join(rnd, "launches_c*.csv")), key=cfgnum):
    rows = list(csv.reader(open(p)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    iK, iM, iV, iU = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    acc = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter(); ids = set()
    for r in rows[hi + 1:]:
        if len(r) <= iV or r[iK].startswith("void at::"):
            continue
        name = r[iK].split("(")[0].replace("void ", "").replace("mci::", "")
        acc[name][r[iM]] += float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1)
        if (r[0], name) not in ids:
            ids.add((r[0], name)); cnt[name] += 1
    for name, m in acc.items():
        n = cnt[name]
        print(f"| {cfgnum(p)} | `{name}` | {n} | {m['gpu__time_duration.sum'] / n:.1f} | {m['dram__bytes_read.sum'] / n / 1e6:.1f} | "
              f"{m['dram__bytes_write.sum'] / n / 1e6:.1f} | {m['smsp__inst_executed.sum'] / n / 1e6:.1f} |")
if reports:
    print("\n## Key counters of the dominant kernels (full captures)\n")
    here = os.path.dirname(os.path.abspath(__file__))
    for label, rep in reports:
        out = subprocess.run([sys.executable, os.path.join(here, "ncu_keys.py"), rep], capture_output=True, text=True).stdout
        print(out.replace(rep, label))
print("\n## Bench lines (default `bench.py --config c`)\n")
print("| config | ms / step | roofline frac | bound | parity max | e2e (samples/s) | clocks |")
print("|---|---|---|---|---|---|---|")
def bnum(p): return int(re.search(r"bench_c(\d+)\.json", p).group(1))
for p in sorted([q for q in glob.glob(os.path.join(rnd, "bench_c*.json")) if re.search(r"bench_c\d+\.json$", q)], key=bnum):
    d = json.load(open(p))
    par = (d.get("parity") or {}).get("max_rel_l2")
    e2e = (d.get("e2e") or {}).get("value")
    print(f"| {bnum(p)} | {d['ms_per_step']:.4f} | {d['roofline']['frac']:.3f} | {d['roofline']['bound']} | {par:.2e} | "
          f"{e2e:.3e} | {d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']} |")
