# 4-GPU measurement survey (scratch recipe): tables, C9 multicast split sweep, C3 / C8 timelines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/gpu.sh table 4 c3 c8 c12 c2 c5
for k in 0 9 5 3; do
  LLRL_MC_UNICAST_PERIOD=$k timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port $((29600 + k)) bench.py --gpus 4 --config c9 --multicast --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/c9mc_$k.err | tail -1 > gpurun_out/c9mc_$k.json
  python -c "import json;d=json.loads(open('gpurun_out/c9mc_$k.json').read());print('c9 mc period=$k', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['reasons'])"
done
bash tools/gpu.sh timeline 4 c3; cat gpurun_out/timeline_c3_n4.jsonl | tail -8
bash tools/gpu.sh timeline 4 c8; cat gpurun_out/timeline_c8_n4.jsonl | tail -8
