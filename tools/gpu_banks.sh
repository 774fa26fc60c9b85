#!/bin/bash
# parity of the fp64 DMMA kernels + their timing + per-instruction bank tables after a layout change
set -u
TAG=${TAG:-r02bk}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "${TESTK:-float64 or f64 or D1 or D2 or C64 or fuzz or dist}" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-subconfigs"
for c in ${CFGS:-C64 D1 D2}; do
  $B --config $c > $O/b_$c.json 2> $O/b_$c.err
  python -c "import json;d=json.loads(open('$O/b_$c.json').read().strip().splitlines()[-1]);print('$c', d['ms_per_step'], d['pass_ms'], d['roofline']['frac'])" || tail -3 $O/b_$c.err
done
P="python bench.py --steps 3 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs"
for spec in ${NCUS:-C64:dmma2 D1:kron_dmma_kernel D2:dmma2g}; do
  n=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 --launch-count 1 -o $O/ncu_$n $P --config $n > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py $O/ncu_$n.ncu-rep $n $O/ncu_$n.json > /dev/null 2>&1
  python tools/ncu_bank_table.py $O/ncu_$n.ncu-rep $O/banks_$n.json 30
  rm -f $O/ncu_$n.ncu-rep
done
