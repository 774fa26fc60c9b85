#!/bin/bash
# chain kernel: parity (chain / fuzz / odd-P tests) and Table 4 #17 / #19 timings
O=gpurun_out/${TAG:-r02ch2}; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "chain or fuzz or odd or table" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
grep -E "^E |FAILED" $O/pytest.log | head -10
timeout 600 python bench.py --sweep table4 --steps 20 --warmup 5 > $O/table4.jsonl 2> $O/table4.err
python - $O/table4.jsonl <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    if d.get('id') in (17, 19, 20, 21): print('t4', d['id'], d['plan'], d.get('ms'), d.get('hbm_gbs'), d.get('graph_ms'))
PY
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${NCUK:-chain_kernel}" -c 2 -o $O/ncu python bench.py --sweep table4 --steps 1 --warmup 3 > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/ncu.ncu-rep x $O/ncu.json > /dev/null 2>&1; git checkout profiles/ncu_traffic.json 2>/dev/null
  python tools/ncu_bank_table.py $O/ncu.ncu-rep $O/banks.json > $O/banks.txt 2>&1; cat $O/banks.txt
  rm -f $O/ncu.ncu-rep
fi
