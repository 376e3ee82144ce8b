# A/B (scratch, 1 GPU): item-outer / chunk-inner role loops (HEAD working tree) vs a80a60a (pre-claims)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _ab/a80a60a && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -x -q -k "toy or edge or guard" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -x -q -k "full" 2>&1 | tail -2
one() {  # label dir cfg
  (cd $2 && timeout 600 python bench.py --config $3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json)
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $3', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  for cfg in c10 c7 c11 c12 c2 c3 c4; do one head . $cfg; done
  for cfg in c10 c11 c2; do one a80a60a _ab/a80a60a $cfg; done
done
LLRL_STATIC_FRAC=0 one head-frac0 . c3
LLRL_STATIC_FRAC=0 one head-frac0 . c10
