python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or mx" > gpurun_out/ai_gpu_tests.log 2>&1; echo pytest rc=$?
for v in 6 7; do for c in c2 c3 c7; do LLRL_CAST_VARIANT=$v python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ai_bench_${c}_v$v.log 2>&1; echo $c v$v rc=$?; done
LLRL_CAST_VARIANT=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2980$v bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e > gpurun_out/ai_bench_c2n2_v$v.log 2>&1; echo c2n2 v$v rc=$?; done
