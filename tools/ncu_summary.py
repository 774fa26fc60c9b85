#!/usr/bin/env python
"""Summarise an `ncu --set full` report (.ncu-rep) into a small JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/r01e/prof_B.ncu-rep B profiles/r01_ncu_B.json

Also records dram read+write bytes per launch in profiles/ncu_traffic.json (bench.py's `traffic`).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_pct_peak",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "us": 1e-6, "ms": 1e-3,
              "ns": 1e-9, "s": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:160]}
        stalls = {}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                d[KEYS[h]] = x * UNIT_SCALE.get(u, 1.0) if u in UNIT_SCALE else x
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    x = float(v)
                except ValueError:
                    continue
                if x >= 0.05:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(x, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            if d.get("duration"):
                d["dram_gbs"] = d["dram_bytes"] / d["duration"] / 1e9
        out.append(d)
    return out


def main():
    rep, cfg, dst = sys.argv[1], sys.argv[2], sys.argv[3]
    s = summarize(rep)
    with open(dst, "w") as f:
        json.dump({"report": os.path.basename(rep), "config": cfg, "launches": s}, f, indent=1)
    tpath = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for d in s:
        m = re.search(r"(kron_[a-z0-9_]+_kernel|sliced_generic_[a-z_]*kernel)", d["kernel"])
        if m and "dram_bytes" in d:
            traffic.setdefault(cfg, {})[m.group(1)] = int(d["dram_bytes"])
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
