#!/usr/bin/env python
"""profiles/ncu_traffic.json from a round's ncu launch lists: DRAM bytes (read + write) of one
whole step = the per-launch means of every MCI kernel of the step, summed (bench.py reads it as
roofline.traffic, labelled with its scope and source).

usage: tools/traffic_from_launches.py <round dir, e.g. profiles/r02>"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def step_bytes(path, steps):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    iK, iM, iV, iU = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot = collections.defaultdict(float)
    inst = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= iV or r[iK].startswith("void at::"):
            continue  # torch's own kernels (input casts, reductions) are not part of the step
        if r[iM] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot[r[iK]] += float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1)
        if r[iM] == "smsp__inst_executed.sum":
            inst += float(r[iV].replace(",", ""))
    return sum(tot.values()) / steps, inst / steps


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
    out = {}
    for c in range(2, 13):
        p = os.path.join(ROOT, rnd, f"launches_c{c}.csv")
        if not os.path.exists(p):
            continue
        # the launch lists run bench.py --steps 3 --warmup 3: six steps under ncu
        b, inst = step_bytes(p, 6)
        out[bench.workload(c)["name"]] = {"bytes": b, "scope": "step (all MCI launches of one step, cold cache)",
                                         "source": f"{rnd}/launches_c{c}.csv (ncu dram__bytes_read+write.sum)"}
        if inst:
            out[bench.workload(c)["name"]]["inst"] = inst
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for k, v in out.items():
        print(f"{v['bytes'] / 1e9:8.3f} GB  {k}")


if __name__ == "__main__":
    main()
