#!/usr/bin/env python
"""Per-source-file / per-line breakdown of an ncu --set full report (needs -lineinfo + --import-source):
warp-stall samples, warp instructions and shared-memory wavefronts, from `ncu --page source
--print-source cuda,sass --csv`. Usage: ncu_by_source.py REPORT [top_lines]"""
import csv
import io
import os
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = None
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        d = dict(zip(hdr[2:], r[2:]))  # source-line rows: the aggregated metrics
        yield fname, int(r[0]), r[1], d


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main(rep, top=25):
    per_file, per_line = {}, []
    for f, ln, src, d in rows(rep):
        s, i, w = num(d.get("Warp Stall Sampling (All Samples)")), num(d.get("Instructions Executed")), \
            num(d.get("L1 Wavefronts Shared"))
        a = per_file.setdefault(f, [0.0, 0.0, 0.0])
        a[0] += s; a[1] += i; a[2] += w
        per_line.append((s, i, w, f, ln, src.strip()[:90]))
    T = [sum(v[k] for v in per_file.values()) or 1 for k in range(3)]
    print(f"| file | stall samples | warp instr | smem wavefronts |\n|---|---|---|---|")
    for f, v in sorted(per_file.items(), key=lambda x: -x[1][0]):
        print(f"| {f} | {100*v[0]/T[0]:.1f}% | {100*v[1]/T[1]:.1f}% | {100*v[2]/T[2]:.1f}% |")
    print(f"\ntotals: samples {T[0]:.0f}, warp instr {T[1]:.3e}, smem wavefronts {T[2]:.3e}\n")
    print("| samples | instr | wavefronts | line |\n|---|---|---|---|")
    for s, i, w, f, ln, src in sorted(per_line, reverse=True)[:top]:
        print(f"| {100*s/T[0]:.1f}% | {100*i/T[1]:.1f}% | {100*w/T[2]:.1f}% | {f}:{ln} `{src}` |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
