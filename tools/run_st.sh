# storer depth experiment: 1-GPU configs then 4-GPU configs
for c in c2 c3 c7 c11; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/st_${c}_n1.log 2>&1; done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for c in c2 c3 c5; do timeout 300 $R --master-port 29731 bench.py --gpus 4 --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/st_${c}_n4.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "capped or variants or guard or sweep" > gpurun_out/st_tests.log 2>&1; echo tests rc=$?
