#!/usr/bin/env python
"""Per-source-file SASS opcode mix of an ncu report (warp instructions per unit of work), split by the
pipe class the opcode issues to (ALU vs FMA/fp16 vs LSU vs other). Usage: ncu_pipes.py REPORT UNITS"""
import collections
import csv
import io
import os
import subprocess
import sys

ALU = {'LOP3', 'SHF', 'IADD3', 'ISETP', 'SEL', 'PRMT', 'FLO', 'POPC', 'LEA', 'IABS', 'IMNMX', 'VIMNMX', 'HSETP2',
       'HMNMX2', 'VHMNMX', 'PLOP3', 'BMSK', 'SGXT', 'ISCADD', 'FSEL', 'FSETP', 'P2R', 'R2P', 'BREV', 'VIADD',
       'VIADDMNMX', 'FMNMX', 'CSET', 'CSETP', 'HMNMX', 'LOP'}
FMA = {'IMAD', 'HADD2', 'HFMA2', 'HMUL2', 'FFMA', 'FADD', 'FMUL', 'IDP', 'IMUL', 'I2F', 'F2I'}
LSU = {'LDS', 'STS', 'LDG', 'STG', 'LD', 'ST', 'ATOMS', 'ATOM', 'RED', 'SHFL', 'LDSM', 'UBLKCP', 'LDC'}


def main(rep, units):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = hdr = None
    agg = collections.defaultdict(collections.Counter)
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] != "" or len(r) < 4:
            continue
        d = dict(zip(hdr[2:], r[2:]))
        ins = d.get("Source", "").strip().split()
        if not ins:
            continue
        op = ins[1] if ins[0].startswith('@') and len(ins) > 1 else ins[0]
        try:
            n = float(d.get("Instructions Executed", "0").replace(",", ""))
        except ValueError:
            n = 0.0
        agg[fname][op.split('.')[0]] += n
    print(f"| file | ALU | FMA/fp16 | LSU | other | total |  (warp instructions per unit, {units} units)")
    print("|---|---|---|---|---|---|")
    tot = collections.Counter()
    for f, c in sorted(agg.items(), key=lambda x: -sum(x[1].values())):
        a = sum(v for k, v in c.items() if k in ALU)
        m = sum(v for k, v in c.items() if k in FMA)
        l = sum(v for k, v in c.items() if k in LSU)
        t = sum(c.values())
        tot.update(c)
        print(f"| {f} | {a/units:.0f} | {m/units:.0f} | {l/units:.0f} | {(t-a-m-l)/units:.0f} | {t/units:.0f} |")
    print("\ntop opcodes: " + ", ".join(f"{k} {v/units:.0f}" for k, v in tot.most_common(24)))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
