python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or special or c4 or c2" > gpurun_out/gpu_tests_f.log 2>&1; echo pytest rc=$?
LLRL_CAST_VARIANT=6 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tests/mp_worker.py > gpurun_out/f_mp_v6.log 2>&1; echo mp_v6 rc=$?
B="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for c in c2 c3; do for v in 1 6; do LLRL_CAST_VARIANT=$v python bench.py --config $c $B > gpurun_out/f_bench_${c}_v$v.log 2>&1; echo $c v$v rc=$?; done; done
python bench.py --config c4 $B > gpurun_out/f_bench_c4.log 2>&1; echo c4 rc=$?
for v in 1 6; do LLRL_CAST_VARIANT=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2964$v bench.py --gpus 2 $B > gpurun_out/f_bench_c2_n2_v$v.log 2>&1; echo c2n2 v$v rc=$?; done
