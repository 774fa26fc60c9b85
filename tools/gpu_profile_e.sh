#!/bin/bash
# Config E profile set (v11): launch list, one ncu --set full capture per kernel (source-level: bank and stall tables)
set -u
TAG=${TAG:-r02e}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
B="python bench.py --steps 3 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs"
CFG=${CFG:-E}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$CFG.csv $B --config $CFG > /dev/null 2>&1
python tools/launches_summary.py $O/launches_$CFG.csv $O/launches_$CFG.json > $O/launches_$CFG.txt 2>&1; head -8 $O/launches_$CFG.txt
for k in ${KS:-tri_tm pair_tm}; do
  n=${CFG}_$k
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 -o $O/ncu_$n $B --config $CFG > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py $O/ncu_$n.ncu-rep $CFG $O/ncu_$n.json > /dev/null 2>&1
  python tools/ncu_bank_table.py $O/ncu_$n.ncu-rep $O/banks_$n.json 30 > /dev/null 2>&1
  python tools/ncu_stall_table.py $O/ncu_$n.ncu-rep $O/stalls_$n.json 40 > /dev/null 2>&1
  python -c "
import json; d=json.load(open('$O/ncu_$n.json'))['launches'][0]
print('$n', {k:d[k] for k in ['duration','fma_pipe_pct','issue_pct','smem_pct_peak','dram_gbs','registers','smem_bank_conflicts']}, d['stalls_per_issue'])
s=json.load(open('$O/stalls_$n.json')); print(s['by_opcode'])"
done
cp profiles/ncu_traffic.json $O/ncu_traffic.json; git checkout profiles/ncu_traffic.json 2>/dev/null
