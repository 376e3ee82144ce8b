# A/B (scratch, 1 GPU): static / claimed loops with one inlined item body (working tree) vs 0c542d5 vs a80a60a
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in a80a60a 0c542d5; do (cd _ab/$t && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1); done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -x -q -k "toy or edge or guard" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -x -q -k "full and (c10 or c11 or c12 or c2)" 2>&1 | tail -2
one() {  # label dir cfg
  (cd $2 && timeout 600 python bench.py --config $3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json)
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $3', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  for cfg in c10 c7 c11 c2 c3; do one new . $cfg; one 0c542d5 _ab/0c542d5 $cfg; done
  for cfg in c10 c11; do one a80a60a _ab/a80a60a $cfg; done
done
one new . c12
one new . c4
