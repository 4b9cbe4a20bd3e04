"""paper_2512_12904_b200 — batched HQC.PKE.Decrypt on B200 (sm_100a).

The product is the C-ABI library ``libhqcgpu.so`` (include/hqc_gpu.h, sources in csrc/); this
package is its thin ctypes binding (``paper_2512_12904_b200.hqc``) plus the seeded input generator
(``paper_2512_12904_b200.gen``). Importing the package does not load CUDA; calling any compute entry
point without the built library raises.
"""
__all__ = ["hqc", "gen"]
