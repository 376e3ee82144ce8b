# cast-kernel variant sweep on the NVLink-bound configs (4 GPUs)
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for v in 6 7 8; do for c in c3 c5 c8 c2; do
  LLRL_CAST_VARIANT=$v timeout 300 $R --master-port 2970$v bench.py --gpus 4 --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/var4_${c}_v$v.log 2>&1
done; done
