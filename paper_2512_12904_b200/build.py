"""Build libhqcgpu.so in-tree with nvcc for sm_100a (no JIT, no torch extension ABI)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libhqcgpu.so")
SOURCES = ["hqc_gpu.cu", "hqc_l1.cu", "hqc_l3.cu", "hqc_l5.cu"]
DEPS = SOURCES + ["kernels.cuh", "launchers.h", "levels.cuh", "async_copy.cuh", "encrypt.cuh", "gf256.cuh", "stage1.cuh", "seg_plans.cuh", "stage1_tmem.cuh", "stage2.cuh", "stage3.cuh", "keccak.cuh", "kem.cuh", "syndromes.cuh", "exp_timing.cuh", "stage3_warp.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC"]


def nvcc_cmd(out: str, extra: list[str] | None = None) -> list[str]:
    return [NVCC, *FLAGS, "-shared", "-o", out, *[os.path.join(CSRC, s) for s in SOURCES], *(extra or [])]


def _compile_link(out: str, extra: list[str]) -> subprocess.CompletedProcess:
    """One nvcc per translation unit, in parallel (the per-level units take minutes each), then the link."""
    from concurrent.futures import ThreadPoolExecutor

    objs = [f"{out}.{os.path.splitext(s)[0]}.o" for s in SOURCES]
    cmds = [[NVCC, *FLAGS, "-c", "-o", o, os.path.join(CSRC, s), *extra] for s, o in zip(SOURCES, objs)]
    with ThreadPoolExecutor(len(cmds)) as ex:
        rs = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    bad = [r for r in rs if r.returncode != 0]
    if not bad:
        link = subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *objs], capture_output=True, text=True)
        rs.append(link)
        bad = [link] if link.returncode != 0 else []
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    err = "".join(r.stdout + r.stderr for r in rs)
    return subprocess.CompletedProcess(cmds, 1 if bad else 0, "", err)


def build_variant(out: str, defines: list[str]) -> str:
    """Experiment builds (scripts/exp_variants.py) into a separate .so; never used by the product."""
    r = _compile_link(out, [f"-D{d}" for d in defines])
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError("nvcc failed")
    return out


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    so_m = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "hqc_gpu.h")]
    return all(os.path.getmtime(d) <= so_m for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return SO
    tmp = SO + f".tmp{os.getpid()}"
    extra = ["-Xptxas", "-v"] if verbose else []
    r = _compile_link(tmp, extra)
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError("nvcc failed building libhqcgpu.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
