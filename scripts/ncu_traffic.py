#!/usr/bin/env python
"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of the fused decrypt kernel from
one `ncu --set full` capture per level (scripts/gpu_full.sh: prof_kernels.py --only fused, batch 65536),
read by bench.py for the roofline's "traffic" key. Usage: ncu_traffic.py OUT.json REPORT_L1 REPORT_L3 REPORT_L5"""
import csv
import io
import json
import os
import subprocess
import sys


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    d = {k: (u, x) for k, u, x in zip(h, units, v)}

    def val(name):
        u, x = d[name]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(x.replace(",", "")) * scale

    tu, tx = d["gpu__time_duration.sum"]
    ns = float(tx.replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}[tu]
    return dict(kernel=d["Kernel Name"][1], dram_read=val("dram__bytes_read.sum"),
                dram_write=val("dram__bytes_write.sum"), duration_ns=ns)


def main(out, reps, batches=(65536, 65536, 65536)):
    res = {}
    for level, rep, batch in zip((1, 3, 5), reps, batches):
        m = metrics(rep)
        m.update(level=level, batch=batch, bytes_per_decryption=(m["dram_read"] + m["dram_write"]) / batch,
                 report=os.path.basename(rep))
        res[str(level)] = m
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:5], tuple(int(b) for b in sys.argv[5].split(",")) if len(sys.argv) > 5 else
         (65536, 65536, 65536))
