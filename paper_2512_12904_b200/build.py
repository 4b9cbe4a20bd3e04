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
DEPS = SOURCES + ["kernels.cuh", "launchers.h", "levels.cuh", "async_copy.cuh", "encrypt.cuh", "gf256.cuh", "stage1.cuh", "stage1_tmem.cuh", "stage2.cuh", "stage3.cuh", "keccak.cuh", "kem.cuh", "syndromes.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_cmd(out: str, extra: list[str] | None = None) -> list[str]:
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
            "-shared", "-o", out, *[os.path.join(CSRC, s) for s in SOURCES], *(extra or [])]


def build_variant(out: str, defines: list[str]) -> str:
    """Experiment builds (scripts/exp_variants.py) into a separate .so; never used by the product."""
    r = subprocess.run(nvcc_cmd(out, [f"-D{d}" for d in defines]), capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
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
    r = subprocess.run(nvcc_cmd(tmp, extra), capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libhqcgpu.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
