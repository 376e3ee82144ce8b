# remote-first interleaving experiment (LLRL_REMOTE_BIAS), 4 GPUs
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30010
for b in 1.0 1.5 3.0; do for c in c3 c8; do port=$((port + 1))
  LLRL_REMOTE_BIAS=$b timeout 300 $R --master-port $port bench.py --gpus 4 --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bias_${c}_$b.log 2>&1
done; done
