#!/bin/bash
# quick E check: parity tests on the E-shaped kernels, E timing (default plan vs round-1 kernels), optional ncu
TAG=${TAG:-r02x}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "${TESTK:-16 or E or fuzz or dist}" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for m in default ${MASKS:-}; do
  if [ $m = default ]; then unset KRON_KINDS_MASK; else export KRON_KINDS_MASK=$m; fi
  python bench.py --config ${CFG:-E} --steps 20 --warmup 5 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_$m.json 2>$O/b_$m.err
  python -c "import json;d=json.loads(open('$O/b_$m.json').read().strip().splitlines()[-1]);print('$m', d['ms_per_step'], d['pass_ms'], d['config']['kernels'])" || tail -3 $O/b_$m.err
done
unset KRON_KINDS_MASK
if [ -n "${NCUK:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCUK -c 1 -o $O/ncu python bench.py --config ${CFG:-E} --steps 2 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/ncu.ncu-rep x $O/ncu.json > /dev/null 2>&1; git checkout profiles/ncu_traffic.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/ncu.json'))['launches'][0]
print({k:d[k] for k in ['duration','fma_pipe_pct','issue_pct','smem_pct_peak','dram_gbs','registers']}, d['stalls_per_issue'])"
fi
