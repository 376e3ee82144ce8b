# bigger / smaller TMA stages for the plain cast path (1 GPU)
for v in 6 9 10; do for c in c2 c3 c7; do
  LLRL_CAST_VARIANT=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var2_${c}_v$v.log 2>&1
done; done
LLRL_CAST_VARIANT=9 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sweep or edge or odd or guard" > gpurun_out/var2_t9.log 2>&1; echo t9 rc=$?
LLRL_CAST_VARIANT=10 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sweep or edge or odd or guard" > gpurun_out/var2_t10.log 2>&1; echo t10 rc=$?
