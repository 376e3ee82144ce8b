python -m pytest tests -m gpu -x -q > gpurun_out/l_gpu_tests.log 2>&1; echo pytest rc=$?
for c in c8 c7 c6; do python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29690 bench.py --gpus 4 --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l_bench_${c}_n4.log 2>&1; echo $c n4 rc=$?; done
