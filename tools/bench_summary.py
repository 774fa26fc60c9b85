#!/usr/bin/env python
"""Summarise a bench.py JSON line file (headline + sub-config lines): python tools/bench_summary.py out.json"""
import json
import sys

lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1])
r = d.get("roofline") or {}
print("HEAD", d["config"]["workload"], "value", d["value"], "ms", d["ms_per_step"], "frac", r.get("frac"),
      "dom", r.get("kernel"), r.get("ms_per_launch"), "step_frac", (d.get("step_roofline") or {}).get("frac"),
      "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
if d.get("e2e"):
    print("  e2e", d["e2e"]["value"], d["e2e"]["unit"])
if d.get("cpu_baseline"):
    print("  cpu", d["cpu_baseline"]["value"], d["cpu_baseline"].get("cpu_model"))
for name, c in (d.get("configs") or {}).items():
    rr = c["roofline"]
    print(f"  {name:4s} ms {c['ms_per_step']:.4f} med {c['median_ms']:.4f} min {c['min_ms']:.4f} GF/s {c['value']:.0f} "
          f"dom-frac {rr['frac']} ({rr['bound']}) step-frac {c['step_roofline']['frac']} plan {c['plan']} "
          f"clk {c['clocks'].get('sm_mhz')}")
