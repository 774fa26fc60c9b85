#!/bin/bash
# tcgen05 tensor-core modes: parity tests, C32 / E bench lines per mode, optional ncu of the tc kernel
TAG=${TAG:-r02tc}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "tensor_core or tf32" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
grep -E "Error|error|assert" $O/pytest.log | head -10
for c in C32 E; do for m in 3xtf32 tf32; do
  timeout 300 python bench.py --config $c --mode $m --steps 20 --warmup 5 --no-cpu --no-e2e > $O/b_${c}_$m.json 2>$O/b_${c}_$m.err
  python -c "import json;d=json.loads(open('$O/b_${c}_$m.json').read().strip().splitlines()[-1]);print('$c $m', d['ms_per_step'], d['pass_ms'], d['config']['kernels'], d['roofline']['frac'], d['roofline']['bound'])" || tail -3 $O/b_${c}_$m.err
done; done
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:kron_tc -c 1 -o $O/ncu_tc python bench.py --config C32 --mode 3xtf32 --steps 2 --warmup 3 --no-autotune --no-cpu --no-e2e > $O/ncu.log 2>&1
fi
