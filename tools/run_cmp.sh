# NCCL comparators (transport only, and the pack -> a2a -> unpack pipeline), 2 and 4 GPUs
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29970
for c in c2 c3 c5; do port=$((port + 1)); timeout 400 $R --nproc-per-node 4 --master-port $port bench.py --gpus 4 --config $c --steps 5 --warmup 3 --no-e2e --comparator > gpurun_out/cmp_$c.log 2>&1; done
timeout 400 $R --nproc-per-node 2 --master-port 29980 bench.py --gpus 2 --config c2 --steps 5 --warmup 3 --no-e2e --comparator > gpurun_out/cmp_c2_n2.log 2>&1
