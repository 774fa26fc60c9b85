#!/bin/bash
# E triple investigation: compute-only microbenchmark + one ncu --set full capture (source) of the triple
O=gpurun_out/${TAG:-tri}; mkdir -p $O
./tools/microbench_tri > $O/mb.jsonl 2>&1; cat $O/mb.jsonl
if [ "${NCU:-1}" = "1" ]; then
  bash tools/ncu_one.sh E gemm3c ${TAG:-tri} 0
  python tools/ncu_stall_table.py $O/prof_E.ncu-rep $O/stalls_E.json 60 > /dev/null 2>&1; head -c 3000 $O/stalls_E.json
fi
