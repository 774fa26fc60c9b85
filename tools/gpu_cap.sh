O=gpurun_out/r02cap; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || exit 1
for c in 0 100 74 57 48; do
  KRON_GRID_CAP=$c python bench.py --config E --steps 6 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/b_$c.json 2>$O/b_$c.err
  python -c "import json;d=json.loads(open('$O/b_$c.json').read().strip().splitlines()[-1]);print('cap $c', d['ms_per_step'], d['pass_ms'], d['clocks'])"
done
