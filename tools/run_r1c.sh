python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_c.log 2>&1; echo pytest rc=$?
python bench.py --steps 30 --warmup 3 --e2e-steps 3 > gpurun_out/c_bench_c2_n1.log 2>&1; echo c2n1 rc=$?
for v in 0 1; do LLRL_FP8_VARIANT=$v python bench.py --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c_bench_c4_n1_v$v.log 2>&1; echo c4 v$v rc=$?; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 30 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/c_bench_c2_n2.log 2>&1; echo c2n2 rc=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 2 --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c_bench_c4_n2.log 2>&1; echo c4n2 rc=$?
