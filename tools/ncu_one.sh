#!/bin/bash
# one ncu --set full capture (with source) of the first launch matching $2 in `bench.py --config $1`
# usage: tools/ncu_one.sh <config> <kernel-regex> <tag> [skip]
set -u
CFG=$1; K=$2; TAG=$3; SKIP=${4:-3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o $OUT/prof_$CFG \
  python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > $OUT/ncu_$CFG.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/ncu_$CFG.log
