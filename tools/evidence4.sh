# Multi-GPU evidence at HEAD (4 GPUs): every GPU test (multi-GPU parity at 2 and 4),
# the 4-GPU table of every config, NVLink counters for C8 / C12, the default-bench scale run
cd $GRAFT_REPO_ROOT
git_rev=$(cat .git_rev 2>/dev/null || echo unknown)
echo "commit $git_rev" > gpurun_out/evidence4.txt
bash tools/gpu.sh tests >> gpurun_out/evidence4.txt 2>&1
bash tools/gpu.sh table 4 c2 c3 c4 c5 c6 c7 c8 c10 c11 c12 >> gpurun_out/evidence4.txt 2>&1
for extra in "--multicast" "--step-sync" "--replicate nccl --step-sync"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port $((29700 + RANDOM % 100)) \
     bench.py --gpus 4 --config c9 $extra --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('c9 $extra', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['reasons'])" >> gpurun_out/evidence4.txt 2>&1
  cp /tmp/o.json "gpurun_out/table_c9_n4_$(echo $extra | tr -d ' -').json"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29790 \
   bench.py --gpus 4 --config c4 --placement rotated --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/table_c4rot_n4.json
bash tools/gpu.sh nvlink 4 c8
bash tools/gpu.sh nvlink 4 c12
bash tools/gpu.sh scale 4
echo done >> gpurun_out/evidence4.txt
