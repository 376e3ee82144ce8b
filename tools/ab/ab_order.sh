# A/B (scratch): static item order of the TMA cast launch -- stride vs block, static share
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cast_item_order" 2>&1 | tail -2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29611
one() {  # label n cfg extra...
  local lab=$1 n=$2 cfg=$3; shift 3; port=$((port+1))
  if [ $n = 1 ]; then timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/tmp/err.txt | tail -1 > /tmp/o.json
  else timeout 600 $R --nproc-per-node $n --master-port $port bench.py --gpus $n --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/tmp/err.txt | tail -1 > /tmp/o.json; fi
  python -c "import json;d=json.loads(open('/tmp/o.json').read());r=d['roofline'];print('$lab n=$n $cfg', d['value'], d['ms_min'], r['bound'], r['frac'], r['t_lb_ms'], d.get('nvfp4_supplied_amax',{}).get('value'), d.get('event_floor_us'), d['clocks']['reasons'], d.get('comparator'))" || tail -5 /tmp/err.txt
}
one default 1 c1
for o in "0.9 0" "0.9 1" "1 1" "0 0"; do
  set -- $o
  export LLRL_STATIC_FRAC=$1 LLRL_STATIC_BLOCK=$2
  for cfg in c3 c8 c5 c2; do one "frac=$1,block=$2" 4 $cfg; done
  for cfg in c2 c3 c12; do one "frac=$1,block=$2" 1 $cfg; done
done
unset LLRL_STATIC_FRAC LLRL_STATIC_BLOCK
one comparator 4 c3 --comparator
one comparator 4 c5 --comparator
port=$((port+1))
LLRL_STATIC_BLOCK=1 timeout 600 $R --nproc-per-node 4 --master-port $port tools/timeline.py --gpus 4 --config c8 > gpurun_out/timeline_c8_block.jsonl 2>/dev/null
tail -4 gpurun_out/timeline_c8_block.jsonl
