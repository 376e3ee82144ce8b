# SM-partition experiment (LLRL_SPLIT_SMS = SMs given to the pushes), 4 GPUs
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for sp in 0 24 40 64 96; do for c in c3 c5 c8; do
  LLRL_SPLIT_SMS=$sp timeout 300 $R --master-port 2975$((sp % 10)) bench.py --gpus 4 --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/split_${c}_$sp.log 2>&1
done; done
LLRL_SPLIT_SMS=40 timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/split_tests.log 2>&1; echo tests rc=$?
