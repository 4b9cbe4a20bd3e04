#!/usr/bin/env python
"""Time PKE encrypt / KEM encaps / decaps of an experiment build. Usage: time_kem_lib.py LIB.so LEVELS"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12904_b200 import hqc  # noqa: E402

hqc.LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = [sys.argv[0], "--levels", sys.argv[2], "--iters", "10"]
import prof_kem  # noqa: E402  (scripts/ on sys.path as the script directory)

prof_kem.main()
