# 4 GPUs: per-CTA end spread of the cast launch with every item claimed (the default for
# pushing syncs) on C3 / C8, and the comparators on C8
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/gpu.sh timeline 4 c3; tail -4 gpurun_out/timeline_c3_n4.jsonl
bash tools/gpu.sh timeline 4 c8; tail -4 gpurun_out/timeline_c8_n4.jsonl
timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29877 \
   bench.py --gpus 4 --config c8 --comparator --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_c8_cmp_n4.json
python -c "import json;d=json.loads(open('gpurun_out/bench_c8_cmp_n4.json').read());print(d['value'], d.get('comparator'))"
