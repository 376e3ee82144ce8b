# cast-kernel variant sweep on the quantising and cast configs (1 GPU)
for v in 6 7 8; do for c in c10 c11 c7 c2; do
  LLRL_CAST_VARIANT=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/var_${c}_v$v.log 2>&1
done; done
LLRL_CAST_VARIANT=8 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "odd or edge or guard or special or sweep" > gpurun_out/var_tests.log 2>&1; echo tests rc=$?
