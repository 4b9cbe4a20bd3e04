#!/usr/bin/env python
"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck / initcheck,
one tool per gpurun call). Checks results against the oracle as well."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2512_12904_b200 import hqc  # noqa: E402
from workloads import valid_batch  # noqa: E402


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()


def main():
    B = int(os.environ.get("SAN_B", "70"))
    for level in (1, 3, 5):
        W = valid_batch(level, 123, B)
        p = hqc.params(level)
        ref = oracle.decrypt_batch(W["params"], W["u"], W["v"], W["y"])
        m = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
        hqc.hqc_decrypt_batch(level, d(W["u"]), d(W["v"]), d(W["y"]), m)
        r = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device="cuda")
        hqc.hqc_sparse_dense_mul_batch(level, d(W["u"]), d(W["y"]), d(W["v"]), r)
        s = torch.empty(B * p.n1, dtype=torch.uint8, device="cuda")
        hqc.hqc_rm_decode_batch(level, r, s)
        m3 = torch.empty(B * p.k, dtype=torch.uint8, device="cuda")
        ok = torch.empty(B, dtype=torch.uint8, device="cuda")
        hqc.hqc_rs_decode_batch(level, s, m3, ok)
        torch.cuda.synchronize()
        assert (m.cpu().numpy().reshape(B, p.k) == ref).all(), f"fused L{level}"
        assert (m3.cpu().numpy().reshape(B, p.k) == ref).all(), f"stages L{level}"
        if os.environ.get("SAN_DEC_ONLY"):  # a forced decrypt kernel (HQC_DEC_KERNEL): the rest is the same
            continue
        H = np.zeros((W["h"].shape[0], p.u_stride), np.uint64)
        H[:, : W["h"].shape[1]] = W["h"]
        S = np.zeros_like(H)
        S[:, : W["s"].shape[1]] = W["s"]
        uo = torch.empty(B * p.u_stride * 8, dtype=torch.uint8, device="cuda")
        vo = torch.empty(B * p.v_words * 8, dtype=torch.uint8, device="cuda")
        hqc.hqc_encrypt_batch(level, d(H), d(S), d(W["key"].astype(np.uint32)), d(W["m"]), d(W["r1"]), d(W["r2"]),
                              d(W["e"]), uo, vo)
        so = torch.empty(H.shape[0] * p.u_stride * 8, dtype=torch.uint8, device="cuda")
        hqc.hqc_keygen_batch(level, d(H), d(W["x"]), d(W["x"]), so)  # any supports: exercises the kernel
        torch.cuda.synchronize()
        assert (uo.cpu().numpy().view(np.uint64).reshape(B, -1) == W["u"]).all(), f"encrypt u L{level}"
        hu, hv, hy = (torch.from_numpy(np.ascontiguousarray(W[k]).view(np.uint8)).pin_memory() for k in ("u", "v", "y"))
        hm = torch.zeros(B * p.k, dtype=torch.uint8).pin_memory()
        ws = torch.empty(hqc.hqc_decrypt_host_workspace_bytes(level, 32), dtype=torch.uint8, device="cuda")
        hqc.hqc_decrypt_batch_host(level, hu, hv, hy, hm, ws, 32)
        torch.cuda.synchronize()
        assert (hm.numpy().reshape(B, p.k) == ref).all(), f"host L{level}"
        # serialized-ciphertext host call, one key
        ub = (p.n + 7) // 8
        one = W["key"] == W["key"][0]
        ct = np.concatenate([W["u"][one].view(np.uint8).reshape(int(one.sum()), -1)[:, :ub],
                             W["v"][one].view(np.uint8).reshape(int(one.sum()), -1)], axis=1)
        hct = torch.from_numpy(np.ascontiguousarray(ct).reshape(-1)).pin_memory()
        hm1 = torch.zeros(int(one.sum()) * p.k, dtype=torch.uint8).pin_memory()
        wsc = torch.empty(hqc.hqc_decrypt_ct_host_workspace_bytes(level, 16), dtype=torch.uint8, device="cuda")
        hqc.hqc_decrypt_ct_batch_host(level, hct, None, d(W["y"][np.nonzero(one)[0][:1]]), hm1, wsc, 16)
        torch.cuda.synchronize()
        assert (hm1.numpy().reshape(-1, p.k) == ref[one]).all(), f"ct host L{level}"
        # step a6 in its three methods
        for meth in ("linear", "nibble", "logexp"):
            syn = torch.empty(B * 2 * p.delta, dtype=torch.uint8, device="cuda")
            hqc.hqc_rs_syndromes_batch(level, s, syn, meth)
        # KEM: keygen from seeds, H_pk, encaps, decaps
        nk = 3
        seeds = torch.arange(nk * 32, dtype=torch.uint8, device="cuda")
        kh, kx, ky, ks = (torch.empty(nk * p.u_stride * 8, dtype=torch.uint8, device="cuda"),
                          torch.empty(nk * p.y_stride * 4, dtype=torch.uint8, device="cuda"),
                          torch.empty(nk * p.y_stride * 4, dtype=torch.uint8, device="cuda"),
                          torch.empty(nk * p.u_stride * 8, dtype=torch.uint8, device="cuda"))
        sig, hpk = torch.empty(nk * p.k, dtype=torch.uint8, device="cuda"), torch.empty(nk * 32, dtype=torch.uint8,
                                                                                         device="cuda")
        hqc.hqc_kem_keygen_batch(level, seeds, kh, kx, ky, ks, sig, hpk)
        key = torch.from_numpy((np.arange(B) % nk).astype(np.uint32)).cuda()
        mm = torch.from_numpy(np.ascontiguousarray(W["m"]).reshape(-1)).cuda()
        ku, kv = torch.empty(B * p.u_stride * 8, dtype=torch.uint8, device="cuda"), torch.empty(
            B * p.v_words * 8, dtype=torch.uint8, device="cuda")
        K1, K2, acc = (torch.empty(B * 64, dtype=torch.uint8, device="cuda"),
                       torch.empty(B * 64, dtype=torch.uint8, device="cuda"), torch.empty(B, dtype=torch.uint8,
                                                                                            device="cuda"))
        wk = torch.empty(hqc.hqc_kem_workspace_bytes(level, B), dtype=torch.uint8, device="cuda")
        hqc.hqc_kem_encaps_batch(level, kh, ks, hpk, key, mm, ku, kv, K1, wk)
        hqc.hqc_kem_decaps_batch(level, kh, ks, hpk, sig, key, ky, ku, kv, K2, acc, wk)
        torch.cuda.synchronize()
        assert int(acc.sum()) == B and torch.equal(K1, K2), f"kem L{level}"
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
