python bench.py > gpurun_out/aa_bench_c2_n1.log 2>&1; echo n1 rc=$?
for n in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n --comparator > gpurun_out/aa_bench_c2_n$n.log 2>&1; echo n$n rc=$?; done
for c in c3 c5; do python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29760 bench.py --gpus 4 --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --comparator > gpurun_out/aa_bench_${c}_n4.log 2>&1; echo $c rc=$?; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/aa_ref.log 2>&1; echo ref rc=$?
