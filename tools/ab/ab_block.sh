# A/B (scratch, 1 GPU): static items striped vs one block per CTA (LLRL_STATIC_BLOCK), current kernel
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
one() {  # label cfg
  timeout 600 python bench.py --config $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $2', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  for b in 0 1; do
    for cfg in c12 c11 c10 c7 c2 c3; do LLRL_STATIC_BLOCK=$b one "block=$b" $cfg; done
  done
done
