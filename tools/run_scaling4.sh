python -m pytest tests/test_gpu_multi.py -m gpu -x -q > gpurun_out/gpu_multi4.log 2>&1; echo multi rc=$?
for n in 2 4; do for c in c2 c3 c5 c4; do
  if [ $n = 2 ] && [ $c = c5 ]; then continue; fi
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --config $c --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_${c}_n$n.log 2>&1; echo $c n$n rc=$?
done; done
