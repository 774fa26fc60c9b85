#!/bin/bash
# Round-2 GPU session: build, GPU tests, the default bench line (config E + sub-configs), the reference arm,
# optional ncu launch list.  usage: tools/gpu_r02.sh <tag> [tests=1] [bench=1] [ncu=0]
set -u
TAG=${1:-r02}; TESTS=${2:-1}; BENCH=${3:-1}; NCU=${4:-0}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
if [ "$TESTS" = "1" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -5 $OUT/pytest_gpu.log
fi
if [ "$BENCH" = "1" ]; then
  T0=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench wall $(( $(date +%s) - T0 )) s"
  python tools/bench_summary.py $OUT/bench.json || tail -20 $OUT/bench.err
  timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref.json 2> $OUT/ref.err; tail -c 400 $OUT/ref.json
fi
if [ "$NCU" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_E.csv \
     python bench.py --steps 5 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > /dev/null 2>&1
  python tools/launches_summary.py $OUT/launches_E.csv $OUT/launches_E.json 2>&1 | head -8
fi
