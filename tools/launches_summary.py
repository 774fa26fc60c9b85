#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum` launch list (CSV) per kernel.

    python tools/launches_summary.py gpurun_out/r01p/launches_B.csv profiles/r01_launches_B.json

Per-launch times under ncu are cold-cache and serialised: compare SHARES of the step, not absolutes.
"""
import csv
import io
import json
import re
import sys
from collections import OrderedDict


def main():
    src, dst = sys.argv[1], sys.argv[2]
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"^void ", "", short)
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(
            r["Metric Unit"], 1e-9)
        t = float(r["Metric Value"].replace(",", "")) * scale
        d = per.setdefault(short, {"launches": 0, "total_s": 0.0, "grid": r["Grid Size"], "block": r["Block Size"]})
        d["launches"] += 1
        d["total_s"] += t
    kron = {k: v for k, v in per.items() if "kron" in k or "dist_" in k}
    tot = sum(v["total_s"] for v in kron.values()) or 1.0
    for v in per.values():
        v["mean_us"] = v["total_s"] / v["launches"] * 1e6
    for k, v in kron.items():
        v["share_of_kron_time"] = v["total_s"] / tot
    json.dump({"source": src, "kernels": per}, open(dst, "w"), indent=1)
    for k, v in per.items():
        print(f"{k[:90]:90s} n={v['launches']:4d} mean={v['mean_us']:10.1f}us share={v.get('share_of_kron_time', 0):.3f}")


if __name__ == "__main__":
    main()
