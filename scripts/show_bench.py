#!/usr/bin/env python
"""Print the headline fields of a bench.py JSON line (the last JSON line of a log)."""
import json
import sys

line = [ln for ln in open(sys.argv[1]).read().splitlines() if ln.startswith("{")][-1]
d = json.loads(line)
print("headline", d["value"], d["ms_per_step"], "frac", round(d["roofline"]["frac"], 4), d["config"]["launch"],
      "launches", d["gpu_launches"], "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
c1 = d.get("config1")
if c1:
    print("config1", c1["value"], c1["graph_ms_per_launch"], round(c1["alu_roofline_frac"], 4),
          c1["single_launch_ms"]["median"])
c4 = d.get("config4")
if c4:
    print("config4", c4["value"], round(c4["alu_roofline_frac"], 4), c4["outputs_equal_message_per_quarter"])
for k, v in (d.get("config5") or {}).get("levels", {}).items():
    print("config5", k, v["value"], round(v["alu_roofline_frac"], 4), v["mismatches_vs_message"])
for k, v in (d.get("levels") or {}).items():
    print("level", k, v["value"], round(v["roofline_frac"], 4))
for k, v in (d.get("standalone_product") or {}).items():
    print("s1", k, v["value"], round(v["alu_roofline_frac"], 4), round(v["smem_bound_frac"], 4))
for k, v in (d.get("next_rows") or {}).items():
    print("next", k, {kk: (round(vv["alu_roofline_frac"], 3) if isinstance(vv, dict) else vv) for kk, vv in v.items()})
print("e2e", d["e2e"]["value"], "cpu", (d.get("cpu_baseline") or {}).get("value"))
