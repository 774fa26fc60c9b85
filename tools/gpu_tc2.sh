#!/bin/bash
# tcgen05 pair timing without the autotuner (static plan = tcgen05 kernel) per mode; optional ncu of the tc kernel
TAG=${TAG:-r02tc2}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for m in 3xtf32 tf32; do
  timeout 300 python bench.py --config C32 --mode $m --steps 20 --warmup 5 --no-autotune --no-cpu --no-e2e > $O/b_$m.json 2>$O/b_$m.err
  python -c "import json;d=json.loads(open('$O/b_$m.json').read().strip().splitlines()[-1]);print('C32 $m', d['ms_per_step'], d['pass_ms'], d['config']['kernels'], d['roofline']['frac'], d['roofline']['bound'])" || tail -3 $O/b_$m.err
done
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:kron_tc -c 1 -o $O/ncu_tc python bench.py --config C32 --mode ${NCU} --steps 2 --warmup 3 --no-autotune --no-cpu --no-e2e > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/ncu_tc.ncu-rep x $O/ncu_tc.json > /dev/null 2>&1
  python tools/ncu_stall_table.py $O/ncu_tc.ncu-rep $O/stalls_tc.json 30 > /dev/null 2>&1
  python -c "
import json; d=json.load(open('$O/ncu_tc.json'))['launches'][0]
print({k:d.get(k) for k in ['duration','issue_pct','smem_pct_peak','dram_gbs','registers']}, d['stalls_per_issue'])
s=json.load(open('$O/stalls_tc.json')); print(s['by_opcode'])"
fi
