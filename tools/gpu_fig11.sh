#!/bin/bash
# Fig 11 weak-scaling workloads (P = 64 / 128, N = 4, fp32): parity test, N = 1 bench lines, N = 2 plumbing run
TAG=${TAG:-r02f11}; O=gpurun_out/$TAG; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q -m gpu -k "P6" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for c in W64 W128; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > $O/$c.json 2> $O/$c.err; tail -c 700 $O/$c.json; tail -2 $O/$c.err
done
KRON_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --config W64 --exchange p2p --grid 1x2 --rows 16 --steps 3 --warmup 3 --no-e2e > $O/W64_n2.json 2> $O/W64_n2.err
tail -c 900 $O/W64_n2.json; tail -3 $O/W64_n2.err
