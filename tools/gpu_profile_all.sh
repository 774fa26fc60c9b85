#!/bin/bash
# Full evidence pass: gpu tests, bench lines (all configs), ncu launch lists + one --set full capture per
# dominant kernel.  Writes gpurun_out/<tag>/.
set -u
TAG=${1:-prof}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_B.json 2> $OUT/bench_B.err
for c in C32 C64 D1 D2 E; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref_B.json 2>&1
for c in B C32 C64 D1 D2 E; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv \
     python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:kron_fused -s 6 -c 1 -o $OUT/prof_B \
   python bench.py --config B --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:kron_fused -s 4 -c 1 -o $OUT/prof_C32 \
   python bench.py --config C32 --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:kron_fused -s 4 -c 1 -o $OUT/prof_C64 \
   python bench.py --config C64 --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:kron_ -s 6 -c 1 -o $OUT/prof_D1 \
   python bench.py --config D1 --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:kron_ -s 6 -c 1 -o $OUT/prof_D2 \
   python bench.py --config D2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:kron_fused -s 6 -c 2 -o $OUT/prof_E \
   python bench.py --config E --steps 3 --warmup 3 --no-cpu --no-e2e --no-autotune > /dev/null 2>&1
ls $OUT
