#!/usr/bin/env python
"""Launch-policy sweeps of the fused decrypt, one process, policies switched through the
per-call environment knobs of kernels.cuh: (a) small batches: K4s (k_decrypt_sb) vs the persistent kernels
(HQC_SB_MAX=0), graph steady-state and single-launch latency; (b) large batches: HQC_DEC_SPLIT sizes.
Inputs: uniformly random u, v with seeded key supports (the decrypt is constant-flow)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402


def graph_ms(run, G=32, R=5):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(G):
            run()
    for _ in range(2):
        g.replay()
    return bench._timed_ms(g.replay, R) / G


def single_ms(run, n=20):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat = []
    for _ in range(n):
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        lat.append(e0.elapsed_time(e1))
    return float(np.median(lat))


def small(levels, sizes):
    dev = torch.device("cuda:0")
    for level in levels:
        p = hqc.params(level)
        Bmax = max(sizes)
        u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).to(dev) for a in bench.make_inputs(level, 0, Bmax, p))
        m = torch.empty(Bmax * p.k, dtype=torch.uint8, device=dev)
        for B in sizes:
            uu, vv, yy, mm = (u[: B * p.u_stride * 8], v[: B * p.v_words * 8], y[: B * p.y_stride * 4], m[: B * p.k])
            run = lambda: hqc.hqc_decrypt_batch(level, uu, vv, yy, mm)  # noqa: E731
            row = {"level": level, "B": B}
            for name, sbmax in (("sb", "1000000000"), ("persistent", "0")):
                os.environ["HQC_SB_MAX"] = sbmax
                run()
                torch.cuda.synchronize()
                gms = graph_ms(run)
                row[name] = {"graph_ms": gms, "rate": B / gms * 1e3, "single_ms": single_ms(run),
                             "shape": hqc.hqc_decrypt_launch_shape(level, B)}
            os.environ.pop("HQC_SB_MAX")
            print(json.dumps(row), flush=True)


def split(levels, B, splits):
    dev = torch.device("cuda:0")
    for level in levels:
        p = hqc.params(level)
        u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).to(dev) for a in bench.make_inputs(level, 0, B, p))
        m = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
        run = lambda: hqc.hqc_decrypt_batch(level, u, v, y, m)  # noqa: E731
        for s in splits:
            os.environ["HQC_DEC_SPLIT"] = str(s)
            run()
            ms = bench._timed_ms(run, 3)
            print(json.dumps({"level": level, "B": B, "split": s, "ms": ms, "rate": B / ms * 1e3}), flush=True)
        os.environ.pop("HQC_DEC_SPLIT")
        del u, v, y, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "small":
        small([1, 3, 5], [1, 8, 33, 148, 296, 512, 1024, 1184, 2048, 4096, 8192, 16384])
    elif what == "large":
        small([1, 3, 5], [32768, 65536, 262144])
    elif what == "cross":
        small([1], [16384, 32768, 49152, 65536, 131072])
        small([5], [4096, 8192, 16384, 32768, 65536])
    elif what == "stagger":
        dev = torch.device("cuda:0")
        cases = [tuple(map(int, c.split(":"))) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
            [(3, 65536), (3, 262144), (1, 16384)]
        for level, B in cases:
            p = hqc.params(level)
            u, v, y = (torch.from_numpy(a.view(np.uint8).reshape(-1)).to(dev) for a in bench.make_inputs(level, 0, B, p))
            m = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
            run = lambda: hqc.hqc_decrypt_batch(level, u, v, y, m)  # noqa: E731
            for ns in (0, 250, 500, 1000, 2000, 4000):
                os.environ["HQC_SB_STAGGER"] = str(ns)
                run()
                ms = graph_ms(run) if B <= 16384 else bench._timed_ms(run, 10)
                print(json.dumps({"level": level, "B": B, "stagger_ns": ns, "ms": ms, "rate": B / ms * 1e3}), flush=True)
            os.environ.pop("HQC_SB_STAGGER")
    elif what == "split":
        B = int(sys.argv[2]) if len(sys.argv) > 2 else 4_194_304
        levels = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 3, 5]
        split(levels, B, [0, 32768, 65536, 131072, 262144, 524288, 1048576])
