#!/usr/bin/env python
"""Key counters and the warp-stall breakdown of every kernel in one ncu report.

usage: tools/ncu_keys.py <report.ncu-rep> [...]   (prints a markdown block per kernel launch)"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU wavefronts %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
STALLS = ["barrier", "long_scoreboard", "wait", "math_pipe_throttle", "mio_throttle", "short_scoreboard",
          "selected", "not_selected", "dispatch_stall", "lg_throttle", "no_instruction", "branch_resolving",
          "membar", "sleeping", "tex_throttle", "drain", "misc"]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for vals in rows[2:]:
            d = dict(zip(hdr, vals))
            u = dict(zip(hdr, units))
            print(f"### {rep}: {d.get('Kernel Name', '?')[:110]}")
            for k, name in KEYS:
                if k in d:
                    print(f"- {name}: {d[k]} {u.get(k, '')}")
            tot = 0.0
            st = {}
            for s in STALLS:
                k = f"smsp__average_warp_latency_issue_stalled_{s}.ratio"
                k2 = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
                for kk in (k2, k):
                    if kk in d:
                        try:
                            st[s] = float(d[kk])
                        except ValueError:
                            pass
                        break
            tot = sum(st.values())
            if tot:
                print("- stalls (share of warp-cycles per issue): " + ", ".join(
                    f"{s} {100 * v / tot:.1f}%" for s, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.01))
            print()


if __name__ == "__main__":
    main()
