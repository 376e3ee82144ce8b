cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -x -q -k "toy or edge" 2>&1 | tail -3
LLRL_CAST_TMAP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "toy_parity_sweep or odd" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_70b_every_byte and c12" 2>&1 | tail -2
for rep in 1 2; do
for t in 1 0; do
  for cfg in c12 c11 c3 c4 c2; do
    LLRL_CAST_TMAP=$t timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/tmp/err.txt | tail -1 > /tmp/o.json
    python -c "import json;d=json.loads(open('/tmp/o.json').read());print('tmap=$t $cfg rep=$rep', d['value'], d['ms_min'], d.get('nvfp4_supplied_amax',{}).get('value'), d['clocks']['reasons'])"
  done
done
done
