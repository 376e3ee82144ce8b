# final measured table, 4 GPUs
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="--gpus 4 --steps 5 --warmup 3 --no-e2e"
port=29900
for c in c2 c3 c4 c5 c6 c8 c9 c11; do port=$((port + 1)); timeout 400 $R --master-port $port bench.py $B --config $c > gpurun_out/final4_$c.log 2>&1; done
timeout 400 $R --master-port 29920 bench.py $B --config c9 --multicast > gpurun_out/final4_c9mc.log 2>&1
timeout 400 $R --master-port 29921 bench.py $B --config c2 --comparator > gpurun_out/final4_c2cmp.log 2>&1
