#!/usr/bin/env python
"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into a markdown file under profiles/."""
import csv
import io
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % (active)"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of 64"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for vals in rows[2:]:
        res.append({h: (u, v) for h, u, v in zip(rows[0], rows[1], vals)})
    return res


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    st = []
    for n, x in zip(h, v):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                st.append((float(x.replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1
    return [(n, 100 * s / tot) for s, n in sorted(st, reverse=True)[:8]]


def main(outfile, reps, launches=None):
    lines = ["# ncu summary", ""]
    if launches and os.path.exists(launches):
        rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
        h = rows[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        lines += [f"## Launch list (`{os.path.basename(launches)}`: gpu__time_duration.sum, --clock-control none; "
                  "cold-cache, serialised — compare shares)", "", "| kernel | launches | total us | share | mean us |",
                  "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% | {sum(v)/len(v)/1e3:.1f} |")
        lines.append("")
    for rep in reps:
        lines += [f"## `{os.path.basename(rep)}` (ncu --set full)", ""]
        for k in raw(rep)[:1]:
            lines += ["| metric | value | unit |", "|---|---|---|"]
            for m, label in METRICS:
                if m in k:
                    u, v = k[m]
                    lines.append(f"| {label} (`{m}`) | {v} | {u} |")
            lines.append("")
        lines += ["Top stall reasons (% of PC samples): " +
                  ", ".join(f"{n} {p:.1f}%" for n, p in stalls(rep)), ""]
    open(outfile, "w").write("\n".join(lines) + "\n")
    print(outfile)


if __name__ == "__main__":
    out = sys.argv[1]
    launches = None
    reps = []
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            launches = a
        else:
            reps.append(a)
    main(out, reps, launches)
