#!/usr/bin/env python
"""Per-source-line totals of an ncu report WITHOUT double counting inlined code: every SASS instruction is
attributed to ONE line (the innermost: the first stage*/gf/keccak/kem header that claims it, else the
kernel file), then warp instructions, shared-memory wavefronts and stall samples are summed per line.
Usage: ncu_lines.py REPORT UNITS [TOP]"""
import collections
import csv
import io
import os
import subprocess
import sys

PREF = ("stage1.cuh", "stage2.cuh", "stage3.cuh", "syndromes.cuh", "encrypt.cuh", "keccak.cuh", "kem.cuh",
        "gf256.cuh", "async_copy.cuh", "cuda_fp16.hpp", "sm_32_intrinsics.hpp", "sm_30_intrinsics.hpp")


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def main(rep, units, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = hdr = None
    line = None
    owner = {}   # address -> (rank, file, line, text)
    metrics = {}
    srctext = {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0] != "":
            try:
                line = int(r[0])
                srctext[(fname, line)] = r[1].strip()[:80]
            except ValueError:
                pass
            continue
        d = dict(zip(hdr[2:], r[2:]))
        a = d.get("Address")
        if not a:
            continue
        rank = PREF.index(fname) if fname in PREF else len(PREF)
        if a not in owner or rank < owner[a][0]:
            owner[a] = (rank, fname, line)
        metrics[a] = (num(d.get("Instructions Executed")), num(d.get("L1 Wavefronts Shared")),
                      num(d.get("Warp Stall Sampling (All Samples)")))
    per = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    for a, (_, f, ln) in owner.items():
        m = metrics[a]
        for i in range(3):
            per[(f, ln)][i] += m[i]
    T = [sum(v[i] for v in per.values()) for i in range(3)]
    print(f"totals per unit: warp instr {T[0]/units:.0f}, smem wavefronts {T[1]/units:.0f}; samples {T[2]:.0f}")
    byfile = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    for (f, _), v in per.items():
        for i in range(3):
            byfile[f][i] += v[i]
    print("| file | warp instr / unit | smem wavefronts / unit | stall samples |\n|---|---|---|---|")
    for f, v in sorted(byfile.items(), key=lambda x: -x[1][1]):
        print(f"| {f} | {v[0]/units:.0f} | {v[1]/units:.0f} | {100*v[2]/max(T[2],1):.1f}% |")
    print("\n| line | warp instr / unit | smem wavefronts / unit | samples |\n|---|---|---|---|")
    for (f, ln), v in sorted(per.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| {f}:{ln} `{srctext.get((f, ln), '')}` | {v[0]/units:.0f} | {v[1]/units:.1f} | {100*v[2]/max(T[2],1):.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
