"""Readers for the cited fixtures under tests/golden/ (values printed in PAPER.md / SPEC.md)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def table1():
    """Table I as {level: dict}."""
    out = {}
    with open(os.path.join(GOLDEN, "table1_params.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            lv, n, w, wr, n1, k, d, n2, dp = (int(x) for x in line.split())
            out[lv] = dict(n=n, w=w, wr=wr, n1=n1, k=k, d=d, n2=n2, dprime=dp)
    return out


def printed():
    out = {}
    with open(os.path.join(GOLDEN, "printed_values.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, val = line.split()[:2]
            out[key] = val
    return out
