# A/B (scratch, 1 GPU): stage-filling strided item rows (LLRL_STAGE_FILL) + packed nv_amax stages
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
one() {  # label cfg extra...
  local lab=$1 cfg=$2; shift 2
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());r=d['roofline'];print('$lab $cfg', d['value'], d['ms_min'], r['bound'], r['frac'], r['t_lb_ms'], d.get('nvfp4_supplied_amax',{}).get('value'), d['clocks']['reasons'])" || tail -5 /tmp/err.txt
}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -x -q -k "toy or edge or guard" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_70b_every_byte and (c12 or c3)" 2>&1 | tail -2
for rep in 1 2; do
for f in 1 0; do
  for cfg in c12 c3 c2 c11; do LLRL_STAGE_FILL=$f one "fill=$f" $cfg; done
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:llrl_k_nv_amax -c 2 --csv \
   python bench.py --config c12 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-nv-supplied 2>/dev/null | grep -E "nv_amax" | cut -c1-300
