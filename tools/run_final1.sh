# final measured table, 1 GPU
for c in c2 c3 c4 c7 c10 c11; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final1_$c.log 2>&1; done
