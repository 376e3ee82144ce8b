# 4 GPUs: the item-order rule engaged by default -- C12 / C3 at 4 and 2 GPUs
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 4 2; do
  for cfg in c12 c3; do
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 300 $R --nproc-per-node $n --master-port $((29950 + RANDOM % 40)) bench.py --gpus $n --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > gpurun_out/rule_${cfg}_n$n.json
    python -c "import json;d=json.loads(open('gpurun_out/rule_${cfg}_n$n.json').read());print('n=$n $cfg', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['roofline']['frac'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
  done
done
echo "($(cat .git_rev))"
