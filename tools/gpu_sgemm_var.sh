#!/bin/bash
# sgemm instance experiments: KRON_SGEMM_VAR selects the tile instance (gemm.cu launch_gemm); VARS / CFGS lists
O=gpurun_out/${TAG:-r02sv}; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for cfg in ${CFGS:-W64}; do for v in ${VARS:-0}; do
  KRON_SGEMM_VAR=$v python bench.py --config $cfg --steps 6 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_${cfg}_$v.json 2>$O/b_${cfg}_$v.err
  python -c "import json;d=json.loads(open('$O/b_${cfg}_$v.json').read().strip().splitlines()[-1]);print('$cfg $v', d['ms_per_step'], d['step_roofline'])" || tail -3 $O/b_${cfg}_$v.err
done; done
