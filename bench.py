#!/usr/bin/env python
"""Benchmark: batched HQC.PKE.Decrypt decryptions/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--level 3] [--batch 65536] [--impl ours|reference]

A step = one pass of the whole hot path (stages 1-3, the fused kernel) over the rank's resident batch.
N > 1 runs under torchrun, one process per GPU; each rank owns ciphertexts [rank*B, (rank+1)*B) of
the same seeded workload (weak scaling, no collective in the timed region); time = max over ranks
of the CUDA-event time; rank 0 prints ONE JSON line. See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HQC-1/3/5 PKE decryptions/sec per B200 and 8xB200; fraction of roofline"
CONFIG_SEED = {1: 0xC0F1_0001, 3: 0xC0F1_0002, 5: 0xC0F1_0003}
ADV_SEED = 0xC0F1_0004  # BASELINE configs[3] (tests/workloads.py CONFIG_SEED[4])
WORKLOAD = {1: "configs[0]-shape HQC-1 PKE decrypt", 3: "configs[1] HQC-3 PKE decrypt, batch 65536/GPU",
            5: "configs[2] HQC-5 PKE decrypt"}


def algorithmic_ops(p) -> dict:
    """Integer ops per ciphertext the method itself must do."""
    pairs = p.w * p.n12 // 32
    s1 = pairs * 3 // 2
    s2 = p.n1 * (128 + 896 + 128)
    d = p.delta
    s3 = 3 * (2 * d * p.n1 + 4 * d * (d + 1) + p.n1 * (d + 1) + 2 * d * p.k)
    hbm = (p.n + 7) // 8 + p.n12 // 8 + 2 * p.w + p.k
    return dict(stage1=s1, stage2=s2, stage3=s3, total=s1 + s2 + s3, pairs=pairs, hbm_bytes=hbm,
                abi_bytes=8 * p.u_stride + 8 * p.v_words + 4 * p.y_stride + p.k)


KECCAK_OPS = 4560  # 32-bit ALU ops per Keccak-f[1600] with 3-input LOP3 and funnel shifts


def shake_perms(msg_bytes: int, out_bytes: int) -> int:
    """Keccak-f[1600] calls of SHAKE256 (rate 136) on msg_bytes (tag included) with out_bytes squeezed."""
    return msg_bytes // 136 + 1 + max(0, (out_bytes + 135) // 136 - 1)


def kem_ops(p) -> dict:
    """Algorithmic 32-bit ALU ops per operation of the SURVEY §8(f) rows: Keccak calls
    x KECCAK_OPS, products at 1.5 ops per (index, 32-bit word) pair, the fixed-weight sampler's
    w(w-1)/2 compares at 2 ops each, encoders and comparisons at 1 op per word/byte."""
    ub, vb = (p.n + 7) // 8, p.n12 // 8
    d = p.delta
    sampler = lambda w: 3 * w + w * (w - 1)  # noqa: E731  (map + w(w-1)/2 compares x 2)
    enc = int(1.5 * p.wr * (p.n / 32 + p.n12 / 32)) + 2 * p.k * 2 * d + 4 * p.n1 * p.mult + 2 * p.wr
    theta = shake_perms(32 + p.k + 1, 32) * KECCAK_OPS
    coins = shake_perms(33, 12 * p.wr) * KECCAK_OPS + 3 * sampler(p.wr)
    kdf = shake_perms(p.k + ub + vb + 1, 64) * KECCAK_OPS
    cmp_ = (p.n + 31) // 32 + p.n12 // 32
    hpk = shake_perms(2 * ub + 1, 32) * KECCAK_OPS
    keygen = (shake_perms(33, 64) + shake_perms(33, ub) + shake_perms(33, 8 * p.w + p.k)) * KECCAK_OPS \
        + 2 * sampler(p.w) + int(1.5 * p.w * p.n / 32) + hpk
    dec = algorithmic_ops(p)["total"]
    return {"encrypt": enc, "encaps": theta + coins + enc + kdf, "decaps": dec + theta + coins + enc + cmp_ + kdf,
            "keygen": keygen, "kdf": kdf}


def ncu_traffic(level: int, batch: int):
    """DRAM bytes (read + write) per launch of the fused kernel from the committed ncu --set full capture
    (profiles/ncu_traffic.json, scripts/ncu_traffic.py), scaled from its batch to this launch's batch."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)[str(level)]
    except (OSError, KeyError, ValueError):
        return None, None
    src = f"profiles/ncu_traffic.json: {t['report']} (batch {t['batch']}), dram__bytes_read.sum + dram__bytes_write.sum"
    if batch != t["batch"]:
        src += f", scaled per decryption ({t['bytes_per_decryption']:.0f} B) to batch {batch}"
    return t["bytes_per_decryption"] * batch, src


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled with NVML every ~2 ms while the timed region
    runs (B200_PROFILING.md "clocks DURING the timed region")."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, torch_device):
        self.dev = torch_device
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.nv = None

    def _handle(self):
        import pynvml as nv
        import torch

        nv.nvmlInit()
        pr = torch.cuda.get_device_properties(self.dev)
        try:
            bus = f"{getattr(pr, 'pci_domain_id', 0):08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv, nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv, nv.nvmlDeviceGetHandleByIndex(self.dev.index or 0)

    def __enter__(self):
        try:
            self.nv, self.h = self._handle()
            self.max_mhz = float(self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = set()
        for _, bits in self.samples:
            for name, attr in self.REASONS.items():
                if bits & int(getattr(self.nv, attr, 0)):
                    reasons.add(name)
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "sm_mhz_min": float(min(sm))}


def dist_setup():
    from paper_2512_12904_b200 import dist as hdist

    return hdist.env()


def make_inputs(level: int, i0: int, B: int, p, nthreads=None):
    """Uniformly random u and v with the key's y (config 4's fourth-quarter construction), host arrays
    (--data random). The decrypt path is constant-flow: its speed does not depend on decodability."""
    from paper_2512_12904_b200 import gen

    seed = CONFIG_SEED[level]
    key = gen.key_of(i0, B)
    k0, nk = int(key[0]), int(key[-1] - key[0] + 1)
    y_keys = gen.support(seed, gen.TAG_Y, k0, nk, p.n, p.w, p.y_stride, nthreads)
    y = np.ascontiguousarray(y_keys[key - k0])
    u = gen.dense(seed, gen.TAG_U_RAND, i0, B, p.n, p.u_stride, nthreads)
    v = gen.dense(seed, gen.TAG_V_RAND, i0, B, p.n12, p.v_words, nthreads)
    return u, v, y


def gen_shape(p):
    from paper_2512_12904_b200 import gen

    return gen.Shape(n=p.n, w=p.w, wr=p.wr, n1=p.n1, k=p.k, n2=p.n2, delta=p.delta, u_stride=p.u_stride,
                     v_words=p.v_words, y_stride=p.y_stride, sup_stride=p.e_stride)


def make_valid_workload(level: int, i0: int, B: int, p, dev, chunk: int = 1 << 18, seed: int | None = None):
    """Valid ciphertexts for BASELINE configs[0..2] built on the device: the seeded
    generator draws keys (h, x, y; one keypair per 256 ciphertexts) and per-ciphertext (m, r1, r2, e)
    on the host; the library's keygen/encrypt kernels produce s, u, v.
    Returns device tensors u, v, y (per-ciphertext rows) and m_ref."""
    import torch

    from paper_2512_12904_b200 import gen, hqc

    seed = CONFIG_SEED[level] if seed is None else seed
    sh = gen_shape(p)
    key = gen.key_of(i0, B)
    k0, nk = int(key[0]), int(key[-1] - key[0] + 1)
    h, x, y = gen.key_draws(seed, sh, k0, nk)

    def d(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).to(dev)

    dh = d(h)
    ds = torch.empty(nk * p.u_stride * 8, dtype=torch.uint8, device=dev)
    hqc.hqc_keygen_batch(level, dh, d(x), d(y), ds)
    du = torch.empty((B, p.u_stride * 8), dtype=torch.uint8, device=dev)
    dv = torch.empty((B, p.v_words * 8), dtype=torch.uint8, device=dev)
    dm = torch.empty((B, p.k), dtype=torch.uint8, device=dev)
    for c0 in range(0, B, chunk):
        n = min(chunk, B - c0)
        m, r1, r2, e = gen.ct_draws(seed, sh, i0 + c0, n)
        kidx = (key[c0:c0 + n] - k0).astype(np.uint32)
        dmm = d(m)
        hqc.hqc_encrypt_batch(level, dh, ds, d(kidx), dmm, d(r1), d(r2), d(e), du[c0:c0 + n], dv[c0:c0 + n])
        dm[c0:c0 + n] = dmm.view(n, p.k)
    dy = d(y[key - k0])
    torch.cuda.synchronize(dev)
    return du.view(-1), dv.view(-1), dy, dm.view(-1)


def cpu_baseline(level: int, u, v, y, got, m_ref=None, budget_s: float = 12.0) -> dict:
    """The oracle, as it stands, on this host's cores over a bounded sample of the same inputs; also
    reports, on that sample, how many oracle outputs differ from the GPU's and from the messages."""
    import oracle

    op = oracle.params(level)
    cores = os.cpu_count() or 1
    done, t_total, n = 0, 0.0, max(cores, 64)
    mism = mism_ref = 0
    while t_total < budget_s and done < u.shape[0]:
        n = min(n, u.shape[0] - done)
        sl = slice(done, done + n)
        t0 = time.perf_counter()
        m = oracle.decrypt_batch(op, u[sl], v[sl], y[sl], nthreads=cores)
        t_total += time.perf_counter() - t0
        mism += int((m != got[sl]).any(axis=1).sum())
        if m_ref is not None:
            mism_ref += int((m != m_ref[sl]).any(axis=1).sum())
        done += n
        n *= 2
    # one thread too, on a short prefix of the same sample
    n1 = min(u.shape[0], 256)
    t0 = time.perf_counter()
    oracle.decrypt_batch(op, u[:n1], v[:n1], y[:n1], nthreads=1)
    one = n1 / (time.perf_counter() - t0)
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"value": done / t_total, "unit": "decryptions/s", "cores": cores, "kind": "oracle",
            "sample": f"first {done} ciphertexts of this rank's batch, oracle decrypt on {cores} threads "
                      f"({t_total:.1f} s)",
            "value_1_thread": one, "cpu": model,
            "parity_mismatches_vs_gpu": mism,
            "oracle_vs_message_mismatches": mism_ref if m_ref is not None else None}


def run_reference(args):
    """This tier has no installable reference implementation (/root/reference holds only the paper):
    the reference arm is the oracle, as it stands, on this host's cores, over a bounded sample of the
    same workload (oracle-encrypted valid ciphertexts of the same generator draws)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    import oracle

    from paper_2512_12904_b200 import gen

    op = oracle.params(args.level)
    cores = os.cpu_count() or 1
    per_step = max(4096, cores * 256)  # the same order of sample per thread as the cpu_baseline leg
    sh = gen.Shape(n=op.n, w=op.w, wr=op.wr, n1=op.n1, k=op.k, n2=op.n2, delta=op.delta,
                   u_stride=op.words + (op.words & 1), v_words=op.vwords, y_stride=(op.w + 3) // 4 * 4,
                   sup_stride=(op.wr + 3) // 4 * 4)
    seed = CONFIG_SEED[args.level]
    key = gen.key_of(0, per_step)
    nk = int(key[-1]) + 1
    h, x, y = gen.key_draws(seed, sh, 0, nk)
    s = np.stack([oracle.keygen(op, h[i, : op.words], x[i], y[i]) for i in range(nk)])
    m, r1, r2, e = gen.ct_draws(seed, sh, 0, per_step)
    u, v = oracle.encrypt_batch(op, h, s, key, m, r1, r2, e, nthreads=cores)
    yy = np.ascontiguousarray(y[key])
    for _ in range(args.warmup):
        oracle.decrypt_batch(op, u, v, yy, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        got = oracle.decrypt_batch(op, u, v, yy, nthreads=cores)
    dt = time.perf_counter() - t0
    val = per_step * args.steps / dt
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "decryptions/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32 (GF(2), GF(2^8))",
           "data": "synthetic: seeded valid ciphertexts (generator draws, oracle keygen+encrypt)",
           "config": {"workload": WORKLOAD[args.level] + " (bounded CPU sample)", "level": args.level,
                      "batch_per_step": per_step},
           "mismatches_vs_message": int((got != m).any(axis=1).sum()),
           "cpu_baseline": {"value": val, "unit": "decryptions/s", "cores": cores, "kind": "oracle",
                            "sample": f"{per_step} ciphertexts per step, {args.steps} steps"},
           "e2e": {"value": val, "unit": "decryptions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


SIDE_BATCH = {1: 65536, 3: 65536, 5: 262144}  # configs[0] is 1024 (launch-latency sized); use 65536


def side_levels(args, dev, world, rank, hdist, hqc, skip):
    """The other levels of the metric ("HQC-1/3/5"), same protocol, fewer steps: valid ciphertexts
    (HQC-5 at configs[2]'s batch 262144), K device-timed launches, max over ranks."""
    import torch

    res = {}
    for level in (1, 3, 5):
        if level == skip:
            continue
        p = hqc.params(level)
        B = SIDE_BATCH[level]
        i0, B = hdist.shard(rank, B)
        du, dv, dy, dref = make_valid_workload(level, i0, B, p, dev)
        dm = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
        for _ in range(3):
            hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        torch.cuda.synchronize()
        steps = max(5, args.steps // 2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            hqc.hqc_decrypt_batch(level, du, dv, dy, dm)
        e1.record()
        torch.cuda.synchronize()
        ms = hdist.max_over_ranks(e0.elapsed_time(e1), dev) / steps
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        hqc.hqc_count_mismatch(level, dm, dref, cnt)
        ops = algorithmic_ops(p)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = 64 * sms * float(measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6
        val = world * B / (ms / 1e3)
        res[str(level)] = {"value": val, "unit": "decryptions/s", "batch_per_gpu": B, "ms_per_step": ms,
                           "steps": steps, "roofline_frac": val * ops["total"] / peak / world,
                           "mismatches_vs_message": hdist.sum_over_ranks(cnt)}
        del du, dv, dy, dref, dm
    return res


def next_rows(args, dev, world, rank, hdist, hqc):
    """SURVEY §8(f) rows 1-3 under the same protocol (device-timed, max over ranks, 65,536 rows per GPU, one
    key per 256 ciphertexts): KeyGen from seeds, PKE Encrypt, KEM Encaps and Decaps, each with its rate and
    its fraction of the ALU roofline (kem_ops). Decaps must accept every honest ciphertext with the
    Encaps key."""
    import torch

    from paper_2512_12904_b200 import gen

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = 64 * sms * float(measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6

    def timed(fn, iters):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return hdist.max_over_ranks(e0.elapsed_time(e1), dev) / iters

    def rate(n, ms, ops):
        v = world * n / (ms / 1e3)
        return {"value": v, "ms_per_step": ms, "batch_per_gpu": n, "alu_roofline_frac": v / world * ops / peak,
                "ops_per_op": ops}

    res = {}
    for level in (1, 3, 5):
        p = hqc.params(level)
        B = 65536
        i0, B = hdist.shard(rank, B)
        nk = (B + 255) // 256
        ko = kem_ops(p)

        def d(a):
            return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).to(dev)

        def empty(nbytes):
            return torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)

        # KeyGen is timed on B keys of its own (a batch of B/256 keys would leave most SMs idle); the
        # first nk of them serve the KEM rows below
        seeds = d(gen.rand_bytes(CONFIG_SEED[level], gen.TAG_TEST, i0, B, 32))
        h, x, y, s = (empty(B * p.u_stride * 8), empty(B * p.y_stride * 4), empty(B * p.y_stride * 4),
                      empty(B * p.u_stride * 8))
        sigma, hpk = empty(B * p.k), empty(B * 32)
        kg = timed(lambda: hqc.hqc_kem_keygen_batch(level, seeds, h, x, y, s, sigma, hpk), 3)
        key = d((np.arange(B) // 256).astype(np.uint32))
        m = d(gen.rand_bytes(CONFIG_SEED[level], gen.TAG_TEST, (1 << 24) + i0, B, p.k))
        u, v = empty(B * p.u_stride * 8), empty(B * p.v_words * 8)
        K1, K2, acc = empty(B * 64), empty(B * 64), empty(B)
        ws = empty(hqc.hqc_kem_workspace_bytes(level, B))
        hqc.hqc_kem_encaps_batch(level, h, s, hpk, key, m, u, v, K1, ws)  # key indices range-checked once
        enc = timed(lambda: hqc.hqc_kem_encaps_batch(level, h, s, hpk, key, m, u, v, K1, ws, check_keys=False), 5)
        dec = timed(lambda: hqc.hqc_kem_decaps_batch(level, h, s, hpk, sigma, key, y, u, v, K2, acc, ws,
                                                     check_keys=False), 5)
        ok = int(acc[:B].sum().item()) == B and torch.equal(K1[: B * 64], K2[: B * 64])
        _, r1, r2, e = gen.ct_draws(CONFIG_SEED[level], gen_shape(p), i0, B)  # valid supports
        r1, r2, e = d(r1), d(r2), d(e)
        pke = timed(lambda: hqc.hqc_encrypt_batch(level, h, s, key, m, r1, r2, e, u, v, check_keys=False), 5)
        res[str(level)] = {"keygen_from_seed": rate(B, kg, ko["keygen"]), "pke_encrypt": rate(B, pke, ko["encrypt"]),
                           "kem_encaps": rate(B, enc, ko["encaps"]), "kem_decaps": rate(B, dec, ko["decaps"]),
                           "decaps_accepts_all_and_K_equal": bool(hdist.sum_over_ranks(
                               torch.tensor([0 if ok else 1], device=dev)) == 0)}
        del h, x, y, s, u, v, K1, K2, ws, r1, r2, e
    return res


def standalone_product(args, dev, world, rank, hdist, hqc):
    """BASELINE configs[4] second part: the standalone sparse x dense product (hqc_sparse_dense_mul_batch,
    v = NULL) at (n, w) = (17669, 66), (35851, 100), (57637, 131), against its ALU roofline (1.5 ops
    per (index, 32-bit word) pair) and its HBM traffic (u, y read; r written)."""
    import torch

    res = {}
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = 64 * sms * float(measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6
    for level in (1, 3, 5):
        p = hqc.params(level)
        B = 65536
        i0, B = hdist.shard(rank, B)
        u, _, y = make_inputs(level, i0, B, p)
        du, dy = (torch.from_numpy(a.view(np.uint8)).to(dev) for a in (u, y))
        dr = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device=dev)
        for _ in range(3):
            hqc.hqc_sparse_dense_mul_batch(level, du, dy, None, dr)
        torch.cuda.synchronize()
        steps = max(5, args.steps // 2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            hqc.hqc_sparse_dense_mul_batch(level, du, dy, None, dr)
        e1.record()
        torch.cuda.synchronize()
        ms = hdist.max_over_ranks(e0.elapsed_time(e1), dev) / steps
        ops = algorithmic_ops(p)
        val = world * B / (ms / 1e3)
        nbytes = 8 * p.u_stride + 4 * p.y_stride + 8 * p.v_words
        kern = int(os.environ.get("HQC_S1_KERNEL", "0") or 0)  # the library's choice (kernels.cuh: stage1_kernel)
        kern = kern if kern in (1, 2, 3) else 1
        res[f"n={p.n},w={p.w}"] = {"value": val, "unit": "products/s", "batch_per_gpu": B, "ms_per_step": ms,
                                   "kernel": {1: "k_stage1 (one warp per product, CTA-shared work, windows from shared memory)",
                                              2: "k_stage1p (warp pair, windows from shared memory)",
                                              3: "k_stage1t (windows from tensor memory)"}[kern],
                                   "alu_roofline_frac": val / world * ops["stage1"] / peak,
                                   "hbm_gbs": val / world * nbytes / 1e9,
                                   # one 4-byte shared-memory read per (index, word) pair: the bound of the
                                   # shared-memory kernels (k_stage1t reads its windows from TMEM instead)
                                   "smem_bound_frac": val / world * ops["pairs"] / (peak / 2)}
        del du, dy, dr
    return res


def opt_in_variants():
    """The opt-in tensor-memory kernels (not constant-flow, so not the library's defaults),
    timed in subprocesses because the library reads its kernel switches once per process: the standalone
    product with HQC_S1_KERNEL=3 (k_stage1t) and the fused decrypt with HQC_DEC_KERNEL=4 (k_decrypt_t), on
    the same seeded inputs as the default lines (scripts/time_s1_lib.py, scripts/time_lib.py: 20 launches
    after 3 warm-up launches, CUDA events)."""
    import subprocess

    root = os.path.dirname(os.path.abspath(__file__))
    lib = os.path.join(root, "paper_2512_12904_b200", "libhqcgpu.so")
    res = {"constant_flow": False}
    for key, script, env_kv in (("standalone_product_k_stage1t_ms", "time_s1_lib.py", ("HQC_S1_KERNEL", "3")),
                                ("fused_decrypt_k_decrypt_t_ms", "time_lib.py", ("HQC_DEC_KERNEL", "4"))):
        env = dict(os.environ, **{env_kv[0]: env_kv[1]})
        try:
            r = subprocess.run([sys.executable, os.path.join(root, "scripts", script), lib, "1,3,5"], env=env,
                               capture_output=True, text=True, timeout=300)
            line = r.stdout.strip().splitlines()[-1]
            res[key] = json.loads(line[line.index("{"):])
        except Exception as e:  # a variant that cannot run is reported, not fatal for the bench line
            res[key] = f"unavailable: {type(e).__name__}"
    res["batch_per_gpu"] = 65536
    return res


def _alu_peak(dev) -> float:
    """ALU-pipe peak per GPU in int-ops/s: 64 lanes/clk/SM (K7-measured 63.7) x SMs x sm_max_mhz."""
    import torch

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    return 64 * sms * float(measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6


def _timed_ms(fn, steps: int) -> float:
    """Mean device time of fn() over `steps` back-to-back calls, CUDA events on the current stream."""
    import torch

    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def config1_block(args, dev, world, rank, hdist, hqc, B: int = 1024) -> dict:
    """BASELINE configs[0]: HQC-1, batch 1,024 per GPU (valid ciphertexts). Two numbers (SURVEY §7,
    PAPER.md:237 repeated runs): the steady-state rate of back-to-back launches captured in one CUDA Graph
    (launch overhead amortised), and the latency of ONE launch (CUDA events around a single launch on an
    idle GPU, median of 50), plus the host-side wall time of launch + synchronize."""
    import torch

    level = 1
    p = hqc.params(level)
    du, dv, dy, dref = make_valid_workload(level, rank * B, B, p, dev)
    dm = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
    run = lambda: hqc.hqc_decrypt_batch(level, du, dv, dy, dm)  # noqa: E731
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    lat, wall = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(50):
        t0 = time.perf_counter()
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        wall.append(time.perf_counter() - t0)
        lat.append(e0.elapsed_time(e1))
    # one launch captured alone in a graph, replayed with events around each replay: the latency of one
    # batch of 1,024 without the host-side launch cost of a plain stream launch
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1):
        run()
    for _ in range(3):
        g1.replay()
    torch.cuda.synchronize()
    lat_g = []
    for _ in range(50):
        e0.record(st)
        g1.replay()
        e1.record(st)
        e1.synchronize()
        lat_g.append(e0.elapsed_time(e1))
    G, R = 64, 10
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(G):
            run()
    for _ in range(3):
        g.replay()
    ms_graph = _timed_ms(g.replay, R) / G
    ms_stream = _timed_ms(run, G)  # plain back-to-back launches on the stream (no graph)
    ms = hdist.max_over_ranks(ms_graph, dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    hqc.hqc_count_mismatch(level, dm, dref, cnt)
    ops = algorithmic_ops(p)["total"]
    val = world * B / (ms / 1e3)
    grid, wpc = hqc.hqc_decrypt_launch_shape(level, B)
    return {"workload": "configs[0] HQC-1 PKE decrypt, batch 1024/GPU", "batch_per_gpu": B,
            "value": val, "unit": "decryptions/s", "graph_ms_per_launch": ms, "graph_launches": G * R,
            "alu_roofline_frac": val / world * ops / _alu_peak(dev),
            "stream_ms_per_launch": hdist.max_over_ranks(ms_stream, dev),
            "single_launch_ms": {"median": float(np.median(lat)), "min": float(min(lat)), "n": len(lat)},
            "single_graph_launch_ms": {"median": float(np.median(lat_g)), "min": float(min(lat_g)), "n": len(lat_g)},
            "single_launch_host_wall_ms": {"median": 1e3 * float(np.median(wall)), "min": 1e3 * float(min(wall))},
            "launch": {"kernel": hqc.KERNEL_NAMES[hqc.hqc_decrypt_launch_kernel(level, B)], "grid": grid,
                       "warps_per_cta": wpc},
            "mismatches_vs_message": hdist.sum_over_ranks(cnt)}


def config4_block(args, dev, world, rank, hdist, hqc, total: int = 1 << 20) -> dict:
    """BASELINE configs[3]: HQC-1 adversarial decrypt, 1,048,576 ciphertexts in four quarters (DESIGN.md §5,
    R#17), split evenly over the ranks: Q0 valid; Q1 valid with delta RM blocks of v randomised; Q2 with
    delta+1..2 delta blocks randomised; Q3 uniformly random u and v with the key's y. The valid ciphertexts
    are built on the device (generator draws -> GPU encrypt), the block patches and the Q3 rows come from
    the same seeded generator as tests/workloads.adversarial_batch (bit-identical inputs; the full-size
    oracle comparison is tests/test_gpu_config4.py). Timed like the headline; the decrypt is constant-flow,
    so the garbage quarters cost the same as the valid one."""
    import torch

    from paper_2512_12904_b200 import gen

    level = 1
    p = hqc.params(level)
    sh = gen_shape(p)
    i0, n = hdist.split_even(total, world, rank)
    du, dv, dy, dref = make_valid_workload(level, i0, n, p, dev, seed=ADV_SEED)
    q = gen.quarter_of(np.arange(i0, i0 + n), total)
    bw = p.n2 // 64
    v3 = dv.view(torch.int64).view(n, p.n1, bw)
    for quarter, (tmin, tmax) in ((1, (p.delta, p.delta)), (2, (p.delta + 1, 2 * p.delta))):
        mask = q == quarter
        if mask.any():
            _, patches = gen.block_patches(i0, n, ADV_SEED + quarter, sh, tmin, tmax, row_mask=mask)
            for rr, b, bits in patches:
                v3[torch.from_numpy(rr).to(dev), torch.from_numpy(b).to(dev)] = torch.from_numpy(
                    bits.view(np.int64)).to(dev)
    idx = np.nonzero(q == 3)[0]
    if idx.size:
        j0, cnt = int(idx[0]), int(idx.size)
        for c0 in range(0, cnt, 1 << 17):
            c = min(1 << 17, cnt - c0)
            uu = gen.dense(ADV_SEED, gen.TAG_U_RAND, i0 + j0 + c0, c, p.n, p.u_stride)
            vv = gen.dense(ADV_SEED, gen.TAG_V_RAND, i0 + j0 + c0, c, p.n12, p.v_words)
            du.view(n, -1)[j0 + c0:j0 + c0 + c] = torch.from_numpy(uu.view(np.uint8)).to(dev)
            dv.view(n, -1)[j0 + c0:j0 + c0 + c] = torch.from_numpy(vv.view(np.uint8)).to(dev)
    dm = torch.empty(n * p.k, dtype=torch.uint8, device=dev)
    run = lambda: hqc.hqc_decrypt_batch(level, du, dv, dy, dm)  # noqa: E731
    for _ in range(3):
        run()
    ms = hdist.max_over_ranks(_timed_ms(run, max(5, args.steps // 4)), dev)
    eq = (dm.view(n, p.k) == dref.view(n, p.k)).all(dim=1).cpu().numpy()
    per_q = {}
    for quarter in range(4):
        sel = q == quarter
        per_q[f"Q{quarter}"] = [hdist.sum_over_ranks(int(eq[sel].sum()), dev), hdist.sum_over_ranks(int(sel.sum()), dev)]
    val = total / (ms / 1e3)
    ops = algorithmic_ops(p)["total"]
    out = {"workload": "configs[3] HQC-1 adversarial decrypt, batch 1048576 (split over GPUs)", "total_batch": total,
           "value": val, "unit": "decryptions/s", "ms_per_step": ms,
           "alu_roofline_frac": val / world * ops / _alu_peak(dev),
           "outputs_equal_message_per_quarter": per_q,
           "q0_mismatches_vs_message": per_q["Q0"][1] - per_q["Q0"][0],
           "parity": "all 1,048,576 rows vs the oracle: tests/test_gpu_config4.py (-m gpu)"}
    del du, dv, dy, dref, dm, v3
    torch.cuda.empty_cache()
    return out


def config5_block(args, dev, world, rank, hdist, hqc, total: int = 4_194_304) -> dict:
    """BASELINE configs[4]: HQC-1, HQC-3 and HQC-5 each at 4,194,304 valid ciphertexts, split evenly and
    contiguously over the N ranks (hdist.split_even: strong scaling; per-index seeding, so the bytes are the
    same for every N). Per level: K launches of this rank's shard between CUDA events, MAX over ranks; the
    mismatch count vs the generator's messages is SUMmed over NCCL; clocks are sampled on every rank during
    its timed region (hdist.scaling_run, the function the gloo test drives)."""
    import torch

    steps = max(3, args.steps // 8)

    def run_shard(level, i0, n):
        p = hqc.params(level)
        du, dv, dy, dref = make_valid_workload(level, i0, n, p, dev)
        dm = torch.empty(n * p.k, dtype=torch.uint8, device=dev)
        run = lambda: hqc.hqc_decrypt_batch(level, du, dv, dy, dm)  # noqa: E731
        run()
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        with ClockSampler(dev) as clk:
            ms = _timed_ms(run, steps)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        hqc.hqc_count_mismatch(level, dm, dref, cnt)
        bad = int(cnt.item())
        del du, dv, dy, dref, dm
        torch.cuda.empty_cache()
        return ms, bad, clk.summary()

    ops = {lv: algorithmic_ops(hqc.params(lv))["total"] for lv in (1, 3, 5)}
    res = hdist.scaling_run((1, 3, 5), total, world, rank, run_shard, ops, _alu_peak(dev), dev)
    n_rank = hdist.split_even(total, world, rank)[1]
    launch = {lv: {"kernel": hqc.KERNEL_NAMES[hqc.hqc_decrypt_launch_kernel(lv, n_rank)],
                   "launches_per_step": hqc.hqc_decrypt_launch_count(lv, n_rank)} for lv in (1, 3, 5)}
    return {"workload": "configs[4] HQC-1/3/5 PKE decrypt, 4194304 each, split evenly over the GPUs",
            "scaling": "strong", "steps": steps, "launch_per_rank": launch, "levels": res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--level", type=int, default=3, choices=[1, 3, 5])
    ap.add_argument("--batch", type=int, default=65536, help="ciphertexts per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--data", default="valid", choices=["valid", "random"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=8192, help="ciphertexts per pipelined chunk of the host call")
    ap.add_argument("--no-levels", action="store_true", help="skip the per-level side measurements")
    ap.add_argument("--no-variants", action="store_true", help="skip the opt-in tensor-memory kernel timings")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs[0]/[3]/[4] blocks")
    ap.add_argument("--config5-total", type=int, default=4_194_304, help="ciphertexts per level in configs[4]")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2512_12904_b200 import dist as hdist
    from paper_2512_12904_b200 import hqc

    world, rank, local = dist_setup()
    # HQC_BENCH_BACKEND=gloo exercises the N > 1 host logic with all ranks on the visible GPU(s) (a check
    # of the multi-rank code path on a one-GPU box; its timings mean nothing). The product run is NCCL.
    backend = os.environ.get("HQC_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's INIT lines (communicator size, ranks, transports) go to the log, so the run shows that NCCL
        # saw all N ranks
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    p = hqc.params(args.level)
    B = args.batch
    i0, B = hdist.shard(rank, B)  # this rank's shard of the seeded workload (weak scaling)
    if args.data == "valid":
        du, dv, dy, dref = make_valid_workload(args.level, i0, B, p, dev)
    else:
        du, dv, dy = (torch.from_numpy(a.view(np.uint8)).to(dev) for a in make_inputs(args.level, i0, B, p))
        dref = None
    dm = torch.empty(B * p.k, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    # ---- timed region: K fused-kernel launches between CUDA events on the launching stream
    for _ in range(args.warmup):
        hqc.hqc_decrypt_batch(args.level, du, dv, dy, dm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            hqc.hqc_decrypt_batch(args.level, du, dv, dy, dm)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = hdist.max_over_ranks(ev0.elapsed_time(ev1), dev)
    value = world * B * args.steps / (ms / 1e3)

    # ---- correctness of the timed outputs: mismatches vs the generator's messages, summed over ranks
    mismatches = None
    if dref is not None:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        hqc.hqc_count_mismatch(args.level, dm, dref, cnt)
        mismatches = hdist.sum_over_ranks(cnt)

    # ---- e2e: the server-side host call (hqc_decrypt_ct_batch_host): pinned serialized ciphertexts
    #      (u bytes || v bytes) and key indices in, m out; the keys' supports are provisioned on the
    #      device once (outside the timed region); the library pipelines H2D, unpacking, the fused kernel
    #      and D2H over two internal streams; every copy is inside the timed region
    from paper_2512_12904_b200 import gen as hgen

    ub = (p.n + 7) // 8
    key_rel = (hgen.key_of(i0, B) - hgen.key_of(i0, 1)[0]).astype(np.uint32)
    first = np.concatenate([[0], np.nonzero(np.diff(key_rel))[0] + 1])
    dykeys = dy.view(B, -1)[torch.from_numpy(first).to(dev)].contiguous().view(-1)
    hct = torch.cat([du.view(B, -1)[:, :ub], dv.view(B, -1)], dim=1).contiguous().view(-1).cpu().pin_memory()
    hkey = torch.from_numpy(key_rel).pin_memory()
    hm = torch.empty(B * p.k, dtype=torch.uint8).pin_memory()
    chunk = min(B, args.e2e_chunk)
    ws = torch.empty(hqc.hqc_decrypt_ct_host_workspace_bytes(args.level, chunk), dtype=torch.uint8, device=dev)
    hqc.hqc_decrypt_ct_batch_host(args.level, hct, hkey, dykeys, hm, ws, chunk)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.e2e_steps):
        hqc.hqc_decrypt_ct_batch_host(args.level, hct, hkey, dykeys, hm, ws, chunk)
    e1.record(stream)
    torch.cuda.synchronize()
    ems = hdist.max_over_ranks(e0.elapsed_time(e1), dev)
    e2e_ok = bool(torch.equal(hm.to(dev), dref)) if dref is not None else None
    # the link bound of this call: pinned host -> device copy bandwidth, measured here on the same buffers
    dbuf = torch.empty(hct.numel(), dtype=torch.uint8, device=dev)
    dbuf.copy_(hct, non_blocking=True)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(3):
        dbuf.copy_(hct, non_blocking=True)
    c1.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = 3 * hct.numel() / (c0.elapsed_time(c1) / 1e3) / 1e9
    del dbuf
    h2d_bytes = int(hct.numel() + hkey.numel() * 4)
    e2e_val = world * B * args.e2e_steps / (ems / 1e3)
    e2e = {"value": e2e_val, "unit": "decryptions/s", "h2d_bytes_per_step": h2d_bytes,
           "d2h_bytes_per_step": int(B * p.k),
           "api": f"hqc_decrypt_ct_batch_host (pinned serialized ciphertexts + key indices, device-resident "
                  f"key supports, chunk {chunk}, 2 internal streams)",
           "outputs_equal_messages": e2e_ok,
           "h2d_gbs_measured": h2d_gbs,
           "link_bound_decryptions_per_s": world * h2d_gbs * 1e9 / (h2d_bytes / B),
           "link_bound_frac": e2e_val / (world * h2d_gbs * 1e9 / (h2d_bytes / B))}
    # the same through the row-layout host call (u, v, y rows per ciphertext: 9,376 B at HQC-3)
    hu, hv, hy = (t.cpu().pin_memory() for t in (du, dv, dy))
    wsr = torch.empty(hqc.hqc_decrypt_host_workspace_bytes(args.level, chunk), dtype=torch.uint8, device=dev)
    hqc.hqc_decrypt_batch_host(args.level, hu, hv, hy, hm, wsr, chunk)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.e2e_steps):
        hqc.hqc_decrypt_batch_host(args.level, hu, hv, hy, hm, wsr, chunk)
    e1.record(stream)
    torch.cuda.synchronize()
    rms = hdist.max_over_ranks(e0.elapsed_time(e1), dev)
    e2e["row_layout_call"] = {"value": world * B * args.e2e_steps / (rms / 1e3), "api": "hqc_decrypt_batch_host",
                              "h2d_bytes_per_step": int(hu.numel() + hv.numel() + hy.numel())}
    del wsr, ws

    ops = algorithmic_ops(p)
    peaks = measured_peaks()
    c = hdist.merge_clocks(hdist.gather_objects(clk.summary()))  # every rank's clocks: min / union
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    kernel_s = ms / 1e3 / args.steps
    achieved = ops["total"] * B / kernel_s / 1e12
    peak = 64 * sms * sm_max * 1e6 / 1e12  # ALU pipe: 64 lanes/clk/SM (K7-measured 63.7)
    traffic, traffic_src = ncu_traffic(args.level, B)
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tintop/s", "frac": achieved / peak,
            "traffic": traffic,
            "traffic_source": traffic_src,
            "peak_source": f"64 ALU lanes/clk/SM x {sms} SMs x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "ops_per_decryption": ops["total"],
            "frac_at_measured_clock": (achieved / (64 * sms * c["sm_mhz"] * 1e6 / 1e12)) if c["sm_mhz"] else None,
            "roofline_decryptions_per_s": peak * 1e12 / ops["total"],
            "hbm_gbs": ops["abi_bytes"] * B / kernel_s / 1e9,
            "hbm_frac": ops["abi_bytes"] * B / kernel_s / 1e9 / float(peaks.get("hbm_gbs", 6538.6)),
            "smem_bound_decryptions_per_s": 32 * sms * sm_max * 1e6 / ops["pairs"]}
    gw = hqc.hqc_decrypt_launch_shape(args.level, B)
    out = {"metric": METRIC, "value": value, "unit": "decryptions/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u8/u32 (GF(2), GF(2^8))",
           "data": ("synthetic: seeded valid ciphertexts (generator draws, GPU keygen+encrypt)" if dref is not None
                    else "synthetic: uniformly random u,v + seeded key supports (constant-flow path)"),
           "mismatches_vs_message": mismatches,
           "config": {"workload": WORKLOAD[args.level], "level": args.level, "batch_per_gpu": B,
                      "global_batch": world * B, "parallelism": f"dp{world}",
                      "l2": f"inputs {ops['abi_bytes'] * B / 2**20:.0f} MiB/GPU > 126 MB L2, no flush needed",
                      "launch": {"kernel": hqc.KERNEL_NAMES[hqc.hqc_decrypt_launch_kernel(args.level, B)],
                                 "grid": gw[0], "warps_per_cta": gw[1],
                                 "launches_per_step": hqc.hqc_decrypt_launch_count(args.level, B)}},
           "roofline": roof, "e2e": e2e, "gpu_launches": args.steps * hqc.hqc_decrypt_launch_count(args.level, B),
           "clocks": {"sm_mhz": c["sm_mhz"], "sm_max_mhz": c["sm_max_mhz"], "reasons": c["reasons"],
                      "samples": c["samples"], "sm_mhz_min": c["sm_mhz_min"],
                      "per_rank_sm_mhz": c["per_rank_sm_mhz"],
                      "source": "NVML on every rank, 2 ms period, timed region only; sm_mhz = slowest rank's median, "
                                "reasons = union over ranks"}}
    # the wide tables first; the per-config / per-level headline blocks LAST in the line (they are what a
    # reader of the log's tail needs)
    tail = {}
    if not args.no_levels:
        out["next_rows"] = next_rows(args, dev, world, rank, hdist, hqc)
    if rank == 0 and world == 1 and not args.no_levels and not args.no_variants:
        out["opt_in_variants"] = opt_in_variants()
    if not args.no_configs:
        tail["config1"] = config1_block(args, dev, world, rank, hdist, hqc)
        tail["config4"] = config4_block(args, dev, world, rank, hdist, hqc)
    if not args.no_levels:
        tail["standalone_product"] = standalone_product(args, dev, world, rank, hdist, hqc)
        tail["levels"] = side_levels(args, dev, world, rank, hdist, hqc, skip=args.level)
    if not args.no_configs:
        tail["config5"] = config5_block(args, dev, world, rank, hdist, hqc, args.config5_total)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        got = hm.numpy().reshape(B, p.k)
        u = hu.numpy().view(np.uint64).reshape(B, -1)
        v = hv.numpy().view(np.uint64).reshape(B, -1)
        y = hy.numpy().view(np.uint32).reshape(B, -1)
        m_ref = dref.cpu().numpy().reshape(B, p.k) if dref is not None else None
        out["cpu_baseline"] = cpu_baseline(args.level, u, v, y, got, m_ref)
    out.update(tail)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
