#!/bin/bash
# A/B timing of config $CFG under several environment settings: tools/gpu_ab.sh "ENV1=a" "ENV2=b ENV3=c" ...
O=gpurun_out/${TAG:-ab}; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
if [ -n "${TESTK:-}" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$TESTK" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; fi
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 300 python bench.py --config ${CFG:-E} --steps ${STEPS:-20} --warmup 5 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_$i.json 2>$O/b_$i.err
  python -c "import json;d=json.loads(open('$O/b_$i.json').read().strip().splitlines()[-1]);print('$e', d['ms_per_step'], d['pass_ms'], d['config']['kernels'], d['clocks']['sm_mhz'])" || tail -5 $O/b_$i.err
done
