# default bench at 1, 2 and 4 GPUs (what the driver's scaling run does, up to 4)
timeout 600 python bench.py > gpurun_out/scale_n1.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29931 bench.py --gpus 2 > gpurun_out/scale_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29932 bench.py --gpus 4 > gpurun_out/scale_n4.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29933 bench.py --gpus 4 --impl reference > gpurun_out/scale_ref_n4.log 2>&1
