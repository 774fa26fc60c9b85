#!/bin/bash
# Round-2 bench set: default line (E + sub-configs), reference arm, tensor-core mode lines, paper sweeps
set -u
TAG=${TAG:-r02b}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
python tools/bench_summary.py $O/bench_default.json
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
for c in C32 E; do for m in tf32 3xtf32; do
  python bench.py --config $c --mode $m --steps 20 --warmup 5 --no-cpu > $O/bench_${c}_$m.json 2> $O/bench_${c}_$m.err
  python -c "import json;d=json.loads(open('$O/bench_${c}_$m.json').read().strip().splitlines()[-1]);print('$c $m', d['ms_per_step'], d['pass_ms'], d['config']['kernels'], d['roofline']['frac'], d['roofline']['bound'], d['roofline']['peak'])"
done; done
python bench.py --sweep table3 --steps 20 --warmup 5 > $O/table3.jsonl 2> $O/table3.err
python bench.py --sweep table4 --steps 20 --warmup 5 > $O/table4.jsonl 2> $O/table4.err
wc -l $O/table3.jsonl $O/table4.jsonl
