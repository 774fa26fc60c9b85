python __graft_entry__.py > /dev/null 2>&1
timeout 300 python bench.py --dist --config E --steps 3 --warmup 3 2>&1 | tail -2 | cut -c1-600
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-400
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
