#!/usr/bin/env python
"""Join an ncu source-page CSV (--page source --csv --print-source sass) with nvdisasm -g line
annotations of the same kernel: dynamic warp-instruction counts per source line and opcode class.
usage: sass_lines.py <ncu_src.csv> <nvdisasm -g -c output> <mangled kernel name> [csrc file filter]"""
import collections
import csv
import re
import sys

ncu_csv, dis, kern = sys.argv[1:4]
rows = list(csv.reader(open(ncu_csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
dyn = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    dyn.append((r[ix["Source"]], float(r[ix["Instructions Executed"]] or 0), float(r[ix["# Samples"]] or 0)))
# disassembly of the kernel
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
cur = ("?", 0)
stat = []
for l in lines[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l)
    if m:
        stat.append((int(m.group(1), 16), m.group(3), cur))
print("static", len(stat), "dynamic rows", len(dyn), file=sys.stderr)
assert len(stat) == len(dyn), "instruction count mismatch"
CLASS = {"FFMA2": "fp2", "FADD2": "fp2", "FMUL2": "fp2", "LDS": "lds", "STS": "sts", "MOV": "mov", "LOP3": "int",
         "LEA": "int", "IADD3": "int", "IMAD": "int", "SHF": "int", "ISETP": "int", "BRA": "bra", "SYNCS": "sync"}
per = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for (addr, op, loc), (src, n, s) in zip(stat, dyn):
    c = CLASS.get(op, "other")
    per[loc][c] += n
    per[loc]["samples"] += s
    tot[c] += n
ROWS = float(sys.argv[4]) if len(sys.argv) > 4 else 65536.0
print("per row totals:", {k: round(v / ROWS, 1) for k, v in tot.items()})
cols = ["fp2", "lds", "sts", "mov", "int", "bra", "sync", "other", "samples"]
print("%-22s" % "file:line" + "".join("%9s" % c for c in cols))
for loc in sorted(per, key=lambda k: (k[0], k[1])):
    v = per[loc]
    if sum(v[c] for c in cols[:-1]) / ROWS < 4:
        continue
    print("%-22s" % f"{loc[0]}:{loc[1]}" + "".join("%9.1f" % (v[c] / (ROWS if c != "samples" else 1)) for c in cols))
