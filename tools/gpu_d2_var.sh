#!/bin/bash
# D2 experiments: v7 warp counts (KRON_V7_VAR) and the all-GEMM plan (v7 off: KRON_KINDS_MASK=FF7F)
O=gpurun_out/${TAG:-r02d2}; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
[ -n "${TESTK:-}" ] && { timeout 900 python -m pytest tests -x -q -m gpu -k "$TESTK" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; }
for v in ${VARS:-0 1 2 3 4 m}; do
  if [ $v = m ]; then export KRON_KINDS_MASK=FF7F; unset KRON_V7_VAR; else unset KRON_KINDS_MASK; export KRON_V7_VAR=$v; fi
  python bench.py --config D2 --steps 30 --warmup 5 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_$v.json 2>$O/b_$v.err
  python -c "import json;d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]);print('D2 $v', d['ms_per_step'], d['step_stats']['median_ms'], d['pass_ms'], d['config']['kernels'])" || tail -3 $O/b_$v.err
done
