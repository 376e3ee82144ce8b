# fp8 TMA kernel stage / occupancy variants on C4 (1 GPU)
for v in 1 2 3; do LLRL_FP8_VARIANT=$v timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fp8v_$v.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fp8_variants or c4" > gpurun_out/fp8v_tests.log 2>&1; echo tests rc=$?
