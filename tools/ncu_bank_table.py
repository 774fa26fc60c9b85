#!/usr/bin/env python
"""Per-instruction shared-memory wavefront table from an ncu report (source page, SASS view): for every
LDS/STS-class instruction the wavefronts ncu counted, the ideal count (one wavefront per 128 distinct bytes),
the excess, and the N-way conflict degree — to tell real bank conflicts from multi-wavefront vector accesses.

    python tools/ncu_bank_table.py report.ncu-rep out.json [top]
"""
import csv
import io
import json
import subprocess
import sys


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    W, WI, WX = "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive"
    NW, EX, S = "L1 Conflicts Shared N-Way", "Instructions Executed", "Warp Stall Sampling (All Samples)"
    ins = []
    tot = {"wavefronts": 0.0, "ideal": 0.0, "excessive": 0.0, "stall_samples": 0.0}
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        tot["stall_samples"] += num(r[ix[S]]) if S in ix else 0
        w = num(r[ix[W]]) if W in ix else 0
        if w <= 0:
            continue
        wi, wx = num(r[ix[WI]]), num(r[ix[WX]])
        tot["wavefronts"] += w
        tot["ideal"] += wi
        tot["excessive"] += wx
        ins.append({"addr": r[ix["Address"]][-6:], "sass": r[ix["Source"]].strip()[:80], "executed": num(r[ix[EX]]),
                    "wavefronts": w, "ideal": wi, "excessive": wx, "nway": num(r[ix[NW]]) if NW in ix else None})
    ins.sort(key=lambda d: -d["excessive"])
    out = {"report": rep.split("/")[-1], "totals": tot,
           "excess_share": tot["excessive"] / tot["wavefronts"] if tot["wavefronts"] else 0.0,
           "top_excessive": ins[:top]}
    json.dump(out, open(dst, "w"), indent=1)
    print(f"{out['report']}: wavefronts {tot['wavefronts']:.3g} ideal {tot['ideal']:.3g} excessive {tot['excessive']:.3g}"
          f" ({out['excess_share']:.1%})")


if __name__ == "__main__":
    main()
