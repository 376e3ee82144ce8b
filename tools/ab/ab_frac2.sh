# A/B (scratch, 1 GPU): static share of the restructured cast launch on the local-only configs
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
one() {  # label cfg
  timeout 600 python bench.py --config $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-nv-supplied 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $2', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  for f in 1 0.97 0.9; do
    for cfg in c10 c7 c11 c2 c3; do LLRL_STATIC_FRAC=$f one "frac=$f" $cfg; done
  done
done
