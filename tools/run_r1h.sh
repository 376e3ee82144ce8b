python tools/probe_mc.py > gpurun_out/h_probe_mc.log 2>&1; echo probe rc=$?
python -m pytest tests -m gpu -x -q > gpurun_out/h_gpu_tests.log 2>&1; echo pytest rc=$?
for n in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/h_bench_c2_n$n.log 2>&1; echo c2 n$n rc=$?; done
for c in c3 c6; do python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29680 bench.py --gpus 4 --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_bench_${c}_n4.log 2>&1; echo $c n4 rc=$?; done
