#!/usr/bin/env python
"""Build experiment variants of libhqcgpu.so: exp_build.py NAME DEFINE[=V] ... -> scripts/libx_NAME.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12904_b200 import build as b  # noqa: E402

print(b.build_variant(os.path.join(ROOT, "scripts", f"libx_{sys.argv[1]}.so"), sys.argv[2:]))
