# A/B (scratch, 1 GPU): which round-2 commit slowed the quantising cast kernel (C10 MXFP4, C7 MXFP8)?
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in r01 88c1e55 a80a60a e591246 39b238f 6d27aac; do (cd _ab/$t && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1); done
one() {  # label dir cfg
  (cd $2 && timeout 600 python bench.py --config $3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json)
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $3', d['value'], d['ms_min'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for rep in 1 2; do
  for t in r01 88c1e55 a80a60a e591246 39b238f 6d27aac; do one $t _ab/$t c10; done
  one head . c10
done
for t in r01 a80a60a e591246 39b238f; do one $t _ab/$t c7; done
one head . c7
