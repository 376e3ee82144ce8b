cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cast_item_order or cast_variants" 2>&1 | tail -3
for cfg in c4 c2 c3 c12; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$cfg', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['clocks']['reasons'])"
done
