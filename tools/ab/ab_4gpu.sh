# 4-GPU sweep: static vs dynamic claims on the NVLink-bound configs, multicast split periods, timelines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29611
one() {  # label cfg extra...
  local lab=$1 cfg=$2; shift 2; port=$((port+1))
  timeout 600 $R --master-port $port bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());r=d['roofline'];print('$lab $cfg', d['value'], d['ms_min'], r['bound'], r['frac'], r['t_lb_ms'], d.get('nvfp4_supplied_amax',{}).get('value'), d['clocks']['reasons'])" || tail -5 /tmp/err.txt
}
for f in 1 0.9 0.75 0; do
  export LLRL_STATIC_FRAC=$f
  for cfg in c2 c3 c5 c8 c12; do one frac=$f $cfg; done
done
unset LLRL_STATIC_FRAC
for per in 0 9 6 12 4; do
  LLRL_MC_UNICAST_PERIOD=$per one mcper=$per c9 --multicast --step-sync
done
one unicast c9 --step-sync
for f in 1 0.9; do
  port=$((port+1))
  LLRL_STATIC_FRAC=$f timeout 600 $R --master-port $port tools/timeline.py --gpus 4 --config c3 > gpurun_out/timeline_c3_f$f.jsonl 2>/dev/null
  port=$((port+1))
  LLRL_STATIC_FRAC=$f timeout 600 $R --master-port $port tools/timeline.py --gpus 4 --config c8 > gpurun_out/timeline_c8_f$f.jsonl 2>/dev/null
done
