#!/bin/bash
# bench line + ncu launch list + one --set full capture for ONE config: tools/gpu_profile_one.sh <tag> <config> <kernel-regex> <skip> <count>
set -u
TAG=$1; C=$2; K=$3; SK=$4; CN=$5
OUT=gpurun_out/$TAG; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
timeout 300 python bench.py --config $C --steps 30 --warmup 5 --no-cpu > $OUT/bench_$C.json 2> $OUT/bench_$C.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$C.csv \
   python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:$K -s $SK -c $CN -o $OUT/prof_$C \
   python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
ls $OUT
