cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for s in 0 1; do
  for cfg in c2 c3 c4 c11; do
    LLRL_STATIC_ITEMS=$s timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-nv-supplied > gpurun_out/ab_${cfg}_s${s}_r${rep}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_${cfg}_s${s}_r${rep}.json').read().strip().splitlines()[-1]);print('$cfg static=$s rep=$rep', d['value'], d['ms_min'], d['clocks']['reasons'])"
  done
done
done
bash tools/gpu.sh launches c1
bash tools/gpu.sh launches c2
