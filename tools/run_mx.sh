timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "nvfp4 or c11 or mxfp4 or mxfp8 or c10 or c7 or special or edge or guard or odd" > gpurun_out/aq_tests.log 2>&1; echo pytest rc=$?
for c in c11 c10 c7; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/aq_bench_$c.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/aq_launches_c11.csv python bench.py --config c11 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/aq_ncul.log 2>&1; echo ncu rc=$?
