#!/bin/bash
# One GPU session: tests, bench lines for every config, ncu launch list + one full capture.
# usage: tools/gpu_round.sh <tag> [skip_tests]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
if [ "${2:-}" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 300 python bench.py > $OUT/bench_B.json 2> $OUT/bench_B.err; tail -c 3000 $OUT/bench_B.json
for c in C32 C64 D1 D2 E; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  tail -c 600 $OUT/bench_$c.json
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_B.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kron_fused -s 6 -c 1 -o $OUT/prof_B \
   python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_full.log 2>&1
ls -la $OUT
