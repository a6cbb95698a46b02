"""Attribute an ncu capture's warp-stall samples and executed instructions to the
barrier-delimited phases of a kernel (SASS source page), plus the headline pipe
and stall metrics.  Usage: python tools/ncu_phases.py REPORT.ncu-rep [units]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
# one section per captured launch: ["Kernel Name", name] then a header row, then SASS rows
sections, cur_sec = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur_sec = [r[1] if len(r) > 1 else "?", None, []]
        sections.append(cur_sec)
    elif cur_sec is not None and cur_sec[1] is None:
        cur_sec[1] = r
    elif cur_sec is not None:
        cur_sec[2].append(r)
for name, h, body in sections:
    iS, iE, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    seg, cur, tot = [], [0, 0, 0, "start"], 0
    for r in body:
        if len(r) <= max(iS, iE, isrc):
            continue
        s = r[isrc].strip()
        smp, ie = int(r[iS] or 0), int(r[iE] or 0)
        cur[0] += smp; cur[1] += ie; cur[2] += 1; tot += smp
        if s.startswith("BAR") or s.startswith("SYNCS") or "EXIT" in s:
            cur[3] += " | " + s[:34]
            seg.append(cur)
            cur = [0, 0, 0, s[:30]]
    seg.append(cur)
    print("==", name[:100])
    print(f"{'samples':>8} {'winst/unit':>11} {'sass':>5}  phase (closing instruction)")
    for c in seg:
        if c[0] > 0.003 * max(tot, 1):
            print(f"{c[0] / tot * 100:7.1f}% {c[1] / units:11.1f} {c[2]:5d}  {c[3]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hh = r[0]
want = ["gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for v in r[2:]:
    print("== launch", v[hh.index("Kernel Name")][:80] if "Kernel Name" in hh else "")
    for i, n in enumerate(hh):
        if i < len(v) and (n in want or ("stall" in n and n.endswith("per_issue_active.ratio") and float(v[i] or 0) > 0.1)):
            print("  ", n, v[i])
