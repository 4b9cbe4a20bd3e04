#!/usr/bin/env python
"""BASELINE configs[4] on one B200 (the G = 1 shard): 4,194,304 valid ciphertexts per level built on the
device exactly as bench.py builds them, the fused decrypt timed with CUDA events (one launch of the whole
batch per step), every output checked against its generator message."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402


def main(B=4_194_304, steps=5):
    dev = torch.device("cuda:0")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = 64 * sms * float(bench.measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6
    out = {}
    for level in (1, 3, 5):
        p = hqc.params(level)
        du, dv, dy, dref = bench.make_valid_workload(level, 0, B, p, dev)
        dm = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
        hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        hqc.hqc_count_mismatch(level, dm, dref, cnt)
        val = B / (ms / 1e3)
        out[f"HQC-{level}"] = {"batch": B, "ms_per_launch": ms, "decryptions_per_s": val,
                               "alu_roofline_frac": val * bench.algorithmic_ops(p)["total"] / peak,
                               "mismatches_vs_message": int(cnt.item())}
        print(json.dumps({f"HQC-{level}": out[f"HQC-{level}"]}), flush=True)
        del du, dv, dy, dref, dm
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
