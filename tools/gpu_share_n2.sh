#!/bin/bash
# plumbing check of bench.py's N > 1 paths on a one-GPU box: two ranks share cuda:0 (gloo process group)
set -u
OUT=gpurun_out/${1:-share}; mkdir -p $OUT
python __graft_entry__.py > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
export KRON_BENCH_SHARE_GPU=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
# (the default N > 1 line runs config E over NCCL, which cannot put two ranks on one GPU: it refuses with a message)
timeout 600 $R bench.py --gpus 2 --config B --steps 5 --warmup 3 --no-cpu --exchange p2p > $OUT/n2_B.json 2> $OUT/n2_B.err; echo "n2 B rc=$?"; tail -c 700 $OUT/n2_B.json
timeout 600 $R bench.py --gpus 2 --dist --config E --exchange p2p --grid 1x2 --steps 3 --warmup 3 > $OUT/n2_Ep2p.json 2> $OUT/n2_Ep2p.err; echo "n2 E p2p rc=$?"; tail -c 900 $OUT/n2_Ep2p.json
timeout 600 $R bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/n2_ref.json 2> $OUT/n2_ref.err; echo "n2 ref rc=$?"; tail -c 300 $OUT/n2_ref.json
