# A/B (scratch, 4 GPUs): HBM-bound pushing plans (C12) with the local-only item order (0.9 block + claimed tail)
# vs all claimed; parity of that order with remote pushes (mp_worker, no --full)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
LLRL_STATIC_FRAC=0.9 LLRL_STATIC_BLOCK=1 timeout 400 $R --master-port 29901 tests/mp_worker.py 2>&1 | tail -1
one() {  # label cfg
  timeout 300 $R --master-port $((29910 + RANDOM % 80)) bench.py --gpus 4 --config $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $2', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['roofline']['frac'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  one claimed c12
  LLRL_STATIC_FRAC=0.9 LLRL_STATIC_BLOCK=1 one block0.9 c12
done
LLRL_STATIC_FRAC=0.9 LLRL_STATIC_BLOCK=1 one block0.9 c3
