# A/B (scratch, 1 GPU): NVFP4 amax pass with item runs striped over CTAs (LLRL_NV_RUN=32, new default) vs one range per CTA (0)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -q -k "nvfp4 and (toy or guard)" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "full_70b_every_byte and (c11 or c12)" 2>&1 | tail -2
for rep in 1 2; do
  for r in 32 0 128; do
    for cfg in c12 c11; do
      LLRL_NV_RUN=$r timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-nv-supplied 2>/tmp/err.txt | tail -1 > /tmp/o.json
      python -c "import json;d=json.loads(open('/tmp/o.json').read());print('run=$r $cfg', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
    done
  done
done
for r in 32 0; do
  LLRL_NV_RUN=$r timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:llrl_k_nv_amax -c 2 --csv \
     python bench.py --config c12 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-nv-supplied 2>/dev/null | grep nv_amax | awk -F'","' '{print "run='$r' amax ns", $NF}'
done
