# A/B (scratch, 1 GPU): round-1 code (_ab/r01, a git worktree of dd8399c, built in place) vs HEAD
# on the quantising configs (MX / NVFP4 regressed in round 2?)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _ab/r01 && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
one() {  # label dir cfg
  (cd $2 && timeout 600 python bench.py --config $3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json)
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $3', d['value'], d['ms_min'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  for cfg in c7 c10 c11 c2; do one r01 _ab/r01 $cfg; one head . $cfg; done
done
for v in 6 7 8; do LLRL_CAST_VARIANT=$v one "head-v$v" . c7; LLRL_CAST_VARIANT=$v one "r01-v$v" _ab/r01 c7; done
for cfg in c10 c7; do LLRL_STATIC_FRAC=1 one "head-frac1" . $cfg; LLRL_STATIC_FRAC=0 one "head-frac0" . $cfg; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stride_probe tools/stride_probe.cu && timeout 300 /tmp/stride_probe
