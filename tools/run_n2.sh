# knob sweep for the NVLink-bound C2 at 2 GPUs
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --config c2 --steps 5 --warmup 3 --no-e2e"
timeout 300 $R --master-port 29801 $B > gpurun_out/n2_base.log 2>&1
LLRL_CHUNK_ELEMS=65536 timeout 300 $R --master-port 29802 $B > gpurun_out/n2_ch64k.log 2>&1
LLRL_CHUNK_ELEMS=131072 timeout 300 $R --master-port 29803 $B > gpurun_out/n2_ch128k.log 2>&1
LLRL_CHUNK_ELEMS=16384 timeout 300 $R --master-port 29804 $B > gpurun_out/n2_ch16k.log 2>&1
timeout 300 $R --master-port 29805 $B --max-ctas 96 > gpurun_out/n2_cta96.log 2>&1
timeout 300 $R --master-port 29806 $B --max-ctas 120 > gpurun_out/n2_cta120.log 2>&1
LLRL_CAST_VARIANT=1 timeout 300 $R --master-port 29807 $B > gpurun_out/n2_v1.log 2>&1
