#!/bin/bash
# Round-2 profiling session: per config a launch list (gpu__time_duration) and one `ncu --set full` capture of
# the dominant kernel (with source-level counters for the per-instruction bank-conflict tables).
set -u
TAG=${TAG:-r02p}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
B="python bench.py --steps 3 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs"
run() {  # name, bench args, kernel regex
  local n=$1 args=$2 k=$3
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$n.csv $B $args > /dev/null 2>&1
  python tools/launches_summary.py $O/launches_$n.csv $O/launches_$n.json > $O/launches_$n.txt 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 -o $O/ncu_$n $B $args > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py $O/ncu_$n.ncu-rep $n $O/ncu_$n.json > /dev/null 2>&1
  python tools/ncu_bank_table.py $O/ncu_$n.ncu-rep $O/banks_$n.json 30
  rm -f $O/ncu_$n.ncu-rep $O/launches_$n.csv
  echo "== $n"; cat $O/launches_$n.txt | head -6
}
run E "--config E" gemm3c
run E_pair "--config E" gemm2ws
run B "--config B" kron_fused_pipe
run C32 "--config C32" gemm2ws
run C64 "--config C64" dmma2
run D1 "--config D1" kron_dmma_kernel
run D2 "--config D2" dmma2g
run C32_tf32 "--config C32 --mode tf32" kron_tc
run C32_3xtf32 "--config C32 --mode 3xtf32" kron_tc
du -sh $O
