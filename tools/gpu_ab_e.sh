python __graft_entry__.py > /dev/null 2>&1
O=gpurun_out/${TAG:-r02c}; mkdir -p $O
for m in default 7FF; do
  if [ $m = default ]; then unset KRON_KINDS_MASK; else export KRON_KINDS_MASK=$m; fi
  python bench.py --config E --steps 20 --warmup 5 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/E_$m.json 2>$O/E_$m.err
  python -c "import json;d=json.loads(open('$O/E_$m.json').read().strip().splitlines()[-1]);print('$m', d['ms_per_step'], d['pass_ms'])" || tail -3 $O/E_$m.err
done
unset KRON_KINDS_MASK
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm3c -c 1 -o $O/ncu_v10_triple python bench.py --config E --steps 2 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs > $O/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2ws -c 1 -o $O/ncu_v10_pair python bench.py --config E --steps 2 --warmup 3 --no-autotune --no-cpu --no-e2e --no-subconfigs >> $O/ncu.log 2>&1
ls $O
