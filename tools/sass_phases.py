#!/usr/bin/env python
"""Per-phase view of a kernel from an ncu source-page CSV joined with nvdisasm -g output: the kernel is cut
at its BAR instructions; for every segment the dynamic FP32x2 / LDS / STS / other warp-instruction counts
per thread-row and the stall-sample mix.  usage: sass_phases.py <ncu_src.csv> <nvdisasm.sass> <mangled> [rows] [warps/row]"""
import collections, csv, re, sys
ncu_csv, dis, kern = sys.argv[1:4]
ROWS = float(sys.argv[4]) if len(sys.argv) > 4 else 65536.0
WPR = float(sys.argv[5]) if len(sys.argv) > 5 else 4.0
lines = open(dis).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
rows = list(csv.reader(open(ncu_csv))); hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
cur = None; stat = []
for l in lines[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*);", l)
    if m: stat.append((cur, m.group(2).strip()))
data = [r for r in rows[2:] if len(r) >= len(hdr)]
assert len(stat) == len(data), (len(stat), len(data))
seg = 0; acc = collections.defaultdict(collections.Counter); st = collections.defaultdict(collections.Counter); first = {}
for (loc, txt), r in zip(stat, data):
    op = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", txt).group(2)
    if op == "BAR": seg += 1; first[seg] = loc
    n = float(r[ix["Instructions Executed"]] or 0) / ROWS / WPR
    cls = "fp2" if op in ("FFMA2", "FADD2", "FMUL2") else "lds" if op == "LDS" else "sts" if op == "STS" else "oth"
    acc[seg][cls] += n
    for h in stalls:
        v = float(r[ix[h]] or 0)
        if v: st[seg][h[6:]] += v
tot_all = sum(sum(v.values()) for v in st.values())
for k in sorted(acc):
    tot = sum(st[k].values())
    if tot < 0.003 * tot_all: continue
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in st[k].most_common(6))
    print(f"seg {k:2d} line {first.get(k, ('', 0))[1]:4d}  fp2 {acc[k]['fp2']:6.1f} lds {acc[k]['lds']:5.1f} sts {acc[k]['sts']:5.1f} oth {acc[k]['oth']:6.1f}"
          f"  samples {int(tot):6d} ({100 * tot / tot_all:4.1f}%)  {top}")
