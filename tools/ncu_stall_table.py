#!/usr/bin/env python
"""Per-instruction warp-stall samples from an ncu report (source page, SASS view): totals per opcode and the
top instructions, to see where a kernel's time goes (main loop vs epilogue vs barriers).

    python tools/ncu_stall_table.py report.ncu-rep out.json [top]
"""
import collections
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
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    S, SN, EX = "Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed"
    ins, byop = [], collections.Counter()
    total = 0.0
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        smp = num(r[ix[S]]) if S in ix else 0.0
        total += smp
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@") and len(src.split()) > 1:
            op = src.split()[1]
        byop[op.split(".")[0]] += smp
        ins.append({"addr": r[ix["Address"]][-6:], "sass": src[:90], "samples": smp,
                    "not_issued": num(r[ix[SN]]) if SN in ix else None, "executed": num(r[ix[EX]]) if EX in ix else None})
    ins.sort(key=lambda d: -d["samples"])
    out = {"report": rep.split("/")[-1], "total_samples": total,
           "by_opcode": {k: round(v / total, 4) for k, v in byop.most_common(25)} if total else {},
           "top": ins[:top],
           "top_non_fma": [d for d in ins if not d["sass"].split(".")[0].lstrip("@!P0123456789 ").startswith(("FFMA", "DFMA", "DMMA", "HMMA"))][:top]}
    json.dump(out, open(dst, "w"), indent=1)
    print(out["report"], "samples", total, "by opcode:", out["by_opcode"])


if __name__ == "__main__":
    main()
