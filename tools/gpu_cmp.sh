#!/bin/bash
# quick comparison: static-plan bench lines (no autotune) for the given configs; TESTS=1 runs pytest -m gpu first
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
if [ "${TESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_K:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
fi
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e ${AT:---no-autotune} > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); r=d['roofline']; print('$c', d['ms_per_step'],'ms', r['bound'], 'frac', r['frac'], r['ms_per_launch'], 'step_frac', d['step_roofline']['frac'], d['config'].get('plan'), d['config'].get('autotune'), d['clocks'].get('sm_mhz'))" || tail -5 $OUT/bench_$c.err
done
