#!/bin/bash
# fp32 large-P passes: parity of the sgemm cases, Fig 11 workloads (W64 / W128) with the sgemm kernel and with
# the round-1 register-tiled kernel (KRON_KINDS_MASK=7FFF), optional ncu of the sgemm kernel
TAG=${TAG:-r02s}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "${TESTK:-64 or 128 or 48 or 96 or fuzz}" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for cfg in ${CFGS:-W64 W128}; do
  for m in default ${MASKS:-7FFF}; do
    if [ $m = default ]; then unset KRON_KINDS_MASK; else export KRON_KINDS_MASK=$m; fi
    python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_${cfg}_$m.json 2>$O/b_${cfg}_$m.err
    python -c "import json;d=json.loads(open('$O/b_${cfg}_$m.json').read().strip().splitlines()[-1]);print('$cfg $m', d['ms_per_step'], d['pass_ms'], d['roofline']['frac'], d['config']['kernels'])" || tail -3 $O/b_${cfg}_$m.err
  done
done
unset KRON_KINDS_MASK
if [ -n "${NCUK:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCUK -c 1 -o $O/ncu python bench.py --config ${NCUCFG:-W64} --steps 1 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/ncu.ncu-rep x $O/ncu.json > /dev/null 2>&1; git checkout profiles/ncu_traffic.json 2>/dev/null
  python tools/ncu_bank_table.py $O/ncu.ncu-rep $O/banks.json > $O/banks.txt 2>&1
  python -c "
import json; d=json.load(open('$O/ncu.json'))['launches'][0]
print({k:d[k] for k in ['duration','fma_pipe_pct','issue_pct','smem_pct_peak','dram_gbs','registers']}, d['stalls_per_issue'])"
  python tools/ncu_stall_table.py $O/ncu.ncu-rep $O/stalls.json >> $O/banks.txt 2>&1
  rm -f $O/ncu.ncu-rep
fi
