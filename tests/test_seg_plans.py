"""Host-side checks of the segmented product layout (csrc/seg_plans.cuh, stage1.cuh: s1_seg_product;
DESIGN.md §6.1c). No GPU: the committed header is what scripts/gen_segments.py generates, every plan meets
the constraints the kernel relies on, and a word-level model of the lane decomposition (own funnels, the
neighbour's shifted first word, the top pass) reproduces the plain rotate-and-XOR of Eq. 1."""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_2512_12904_b200", "csrc", "seg_plans.cuh")


def plans():
    src = open(HDR).read()
    out = {}
    for m in re.finditer(r"SegPlan<(\d+)> \{\s*static constexpr uint32_t NB = (\d+), LMAX = (\d+), TP = (\d+);"
                         r"\s*static constexpr uint8_t LEN\[32\] = \{([^}]*)\};", src):
        out[int(m.group(1))] = (int(m.group(2)), int(m.group(3)), int(m.group(4)),
                                [int(x) for x in m.group(5).split(",")])
    return out


def test_header_is_generated():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_segments.py")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert r.stdout == open(HDR).read()


def test_plans_cover_every_product_shape():
    # n1*n2/32 (decrypt r, Encrypt v) and floor(n/32) + 1 (Encrypt u, KeyGen s) per level (Table I)
    need = {17664 // 32, 35840 // 32, 57600 // 32, 17669 // 32 + 1, 35851 // 32 + 1, 57637 // 32 + 1}
    assert need <= set(plans())


@pytest.mark.parametrize("nout", sorted(plans()))
def test_plan_constraints(nout):
    nb, lmax, tp, lens = plans()[nout]
    assert len(lens) == 32 and sum(lens) == nb
    assert lmax == -(-nb // 32) and max(lens) == lmax and lmax - min(lens) <= 3
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    assert len(set(int(s) % 32 for s in starts)) == 32  # every load slot hits 32 distinct banks
    if tp == 0:
        assert nb == nout and lens[31] < lmax  # the last lane loads its own neighbour word
    else:
        assert nb + tp - 1 == nout and lens[31] == lmax and tp <= 2


def funnel(lo, hi, s):
    """__funnelshift_r(lo, hi, s): the low 32 bits of (hi:lo) >> (s & 31)."""
    v = ((hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)) >> (s & 31).astype(np.uint64)
    return (v & np.uint64(0xFFFFFFFF)).astype(np.uint32)


@pytest.mark.parametrize("nout", sorted(plans()))
def test_lane_model_matches_rotate_and_xor(nout):
    nb, lmax, tp, lens = plans()[nout]
    rng = np.random.default_rng(nout)
    q0 = nout + 7
    E = rng.integers(0, 2**32, size=q0 + nout + 1, dtype=np.uint64).astype(np.uint32)
    w = 37
    d = rng.integers(0, 32 * q0 + 1, size=w).astype(np.uint32)
    d[:3] = [0, 32 * q0, 31]  # extreme offsets and shifts
    o, s = d >> 5, d & 31
    q = np.arange(nout)
    want = np.zeros(nout, np.uint32)
    for j in range(w):  # plain definition: word q gets bits [32 q + d, 32 q + d + 32) of E
        want ^= funnel(E[o[j] + q], E[o[j] + q + 1], np.full(nout, s[j], np.uint32))
    got = np.zeros(nout, np.uint32)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(int)
    pre = np.zeros(32, np.uint32)
    acc = [np.zeros(lmax, np.uint32) for _ in range(32)]
    zero = np.zeros(1, np.uint32)
    for j in range(w):
        sj = np.array([s[j]], np.uint32)
        for L in range(32):
            st, ln = starts[L], lens[L]
            nload = min(ln + 1, lmax)  # slots 0 .. min(len, LMAX - 1)
            a = [E[o[j] + st + k] for k in range(nload)] + [0] * (lmax + 1 - nload)
            pre[L] ^= funnel(zero, np.array([a[0]], np.uint32), sj)[0]
            for k in range(min(ln, lmax)):
                hi = a[k + 1] if k + 1 < lmax else 0
                acc[L][k] ^= funnel(np.array([a[k]], np.uint32), np.array([hi], np.uint32), sj)[0]
    x = np.zeros(max(tp, 1), np.uint32)
    for j in range(w):
        if tp:
            sj = np.array([s[j]], np.uint32)
            wv = [E[o[j] + nb + i] for i in range(tp)]
            x[0] ^= funnel(zero, np.array([wv[0]], np.uint32), sj)[0]
            for i in range(1, tp):
                x[i] ^= funnel(np.array([wv[i - 1]], np.uint32), np.array([wv[i]], np.uint32), sj)[0]
    for L in range(32):
        if lens[L] == lmax:
            acc[L][lmax - 1] ^= x[0] if L == 31 else pre[L + 1]
        got[starts[L]:starts[L] + lens[L]] = acc[L][:lens[L]]
    for i in range(1, tp):
        got[nb + i - 1] = x[i]
    assert np.array_equal(got, want)
