python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8 or c4 or special" > gpurun_out/gpu_tests_d.log 2>&1; echo pytest rc=$?
for v in 0 1; do LLRL_FP8_VARIANT=$v python bench.py --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d_bench_c4_n1_v$v.log 2>&1; echo c4 v$v rc=$?; done
for ch in 32768 65536 262144 1048576; do LLRL_CHUNK_ELEMS=$ch python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d_bench_c3_ch$ch.log 2>&1; echo c3 ch$ch rc=$?; done
for ch in 32768 262144 1048576; do LLRL_CHUNK_ELEMS=$ch python bench.py --config c2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d_bench_c2_ch$ch.log 2>&1; echo c2 ch$ch rc=$?; done
