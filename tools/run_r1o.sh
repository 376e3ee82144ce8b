python -m pytest tests -m gpu -x -q > gpurun_out/o_gpu_tests.log 2>&1; echo pytest rc=$?
for mc in "" "--multicast"; do python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29710 bench.py --gpus 4 --config c6 --placement colocated $mc --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/o_bench_c6col_n4$mc.log 2>&1; echo c6 $mc rc=$?; done
