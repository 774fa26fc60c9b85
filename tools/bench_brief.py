#!/usr/bin/env python
"""Run bench.py with the given args and print a one-line summary (or the stderr tail on failure).
    python tools/bench_brief.py LABEL --config E --steps 20 --warmup 5 --no-autotune"""
import json
import subprocess
import sys

label, args = sys.argv[1], sys.argv[2:]
res = subprocess.run([sys.executable, "bench.py", "--no-cpu", "--no-e2e"] + args, capture_output=True, text=True)
lines = [l for l in res.stdout.strip().splitlines() if l.startswith("{")]
if not lines:
    print(label, "FAILED rc", res.returncode, res.stderr.strip().splitlines()[-5:])
    sys.exit(0)
d = json.loads(lines[-1])
r = d["roofline"]
print(label, d["config"]["workload"], "ms/step", d["ms_per_step"], "frac", r["frac"], "dom ms", r["ms_per_launch"],
      "step_frac", d["step_roofline"]["frac"], "plan", d["config"].get("plan"), "sm", d["clocks"].get("sm_mhz"))
