# A/B (scratch, 4 GPUs, short): NVLS multicast fed by TMA bulk stores / copy engine (probe), C9 with LLRL_MC_TMA
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mc_bulk_probe tools/mc_bulk_probe.cu -lcuda && timeout 120 /tmp/mc_bulk_probe 4096
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
LLRL_MC_TMA=1 timeout 180 $R --nproc-per-node 4 --master-port 29801 tests/mp_worker.py --mc-only 2>&1 | tail -2
for t in 0 1; do
  LLRL_MC_TMA=$t timeout 180 $R --nproc-per-node 4 --master-port $((29810 + t)) bench.py --gpus 4 --config c9 --multicast --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('mc_tma=$t c9', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
done
NVL_TIMEOUT=240 bash tools/gpu.sh nvlink 4 c12; tail -2 gpurun_out/nvlink_c12_n4.log; grep -c llrl_k_cast gpurun_out/nvlink_c12_n4.csv
timeout 400 $R --nproc-per-node 4 --master-port 29840 tests/mp_worker.py 2>&1 | tail -2
for cfg in c3 c8 c2; do
  timeout 180 $R --nproc-per-node 4 --master-port $((29850 + RANDOM % 50)) bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('n=4 $cfg', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
done
