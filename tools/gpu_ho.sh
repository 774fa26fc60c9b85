#!/bin/bash
# v11 hand-off check: E-shaped parity tests, E timing with / without the hand-off, optional ncu of the new kernels
O=gpurun_out/${TAG:-ho}; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "${TESTK:-16 or E or fuzz}" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for m in ho noho; do
  if [ $m = noho ]; then export KRON_NO_HANDOFF=1; else unset KRON_NO_HANDOFF; fi
  timeout 300 python bench.py --config ${CFG:-E} --steps 20 --warmup 5 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_$m.json 2>$O/b_$m.err
  python -c "import json;d=json.loads(open('$O/b_$m.json').read().strip().splitlines()[-1]);print('$m', d['ms_per_step'], d['pass_ms'], d['config']['kernels'], d['clocks'])" || tail -5 $O/b_$m.err
done
unset KRON_NO_HANDOFF
if [ -n "${NCUK:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCUK -c 1 -o $O/ncu python bench.py --config ${CFG:-E} --steps 2 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/ncu.ncu-rep x $O/ncu.json > /dev/null 2>&1; git checkout profiles/ncu_traffic.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/ncu.json'))['launches'][0]
print({k:d[k] for k in ['kernel','duration','fma_pipe_pct','issue_pct','smem_pct_peak','dram_gbs','registers']}, d['stalls_per_issue'])"
fi
