#!/usr/bin/env python
"""Static SASS opcode histogram of the library's kernels (cuobjdump -sass), to show what the hot loops are
made of (SHF / LOP3 / LDS / UBLKCP / HFMA2 / REDUX ...) without a GPU.
    python scripts/sass_hist.py [regex ...] > profiles/rNN/sass_hist.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2512_12904_b200", "libhqcgpu.so")


def functions(so=SO):
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            funcs[cur].append(m.group(1))
    return funcs


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main(pats):
    funcs = functions()
    dm = demangle(list(funcs))
    print("| kernel | SASS instructions | top opcodes (count) |")
    print("|---|---|---|")
    for f, ops in sorted(funcs.items(), key=lambda kv: dm[kv[0]]):
        name = dm[f]
        if pats and not any(re.search(p, name) for p in pats):
            continue
        base = collections.Counter(o.split(".")[0] for o in ops)
        top = ", ".join(f"{o} {c}" for o, c in base.most_common(14))
        print(f"| `{name.split('(')[0]}` | {len(ops)} | {top} |")


if __name__ == "__main__":
    main(sys.argv[1:])
