#!/bin/bash
# quick GPU iteration: gpu tests (optional), bench for given configs, optional ncu full capture of config $NCU_CFG
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
fi
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json,sys; d=json.load(open('$OUT/bench_$c.json')); r=d['roofline']; print('$c', d['value'], 'GF/s', d['ms_per_step'],'ms', r['bound'], r['achieved'], r['unit'], 'frac', r['frac'], 'step_frac', d['step_roofline']['frac'], d['config'].get('plan'), d['config'].get('autotune'), d['clocks'].get('sm_mhz'))" || tail -5 $OUT/bench_$c.err
done
if [ -n "${NCU_CFG:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-kron_} -s ${NCU_S:-6} -c 1 -o $OUT/prof_$NCU_CFG \
    python bench.py --config $NCU_CFG --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_full.log 2>&1
fi
