# A/B (scratch, 1 GPU): MX / NVFP4 cast variant (7: 16 KiB x 2 CTAs, the default; 8: 32 KiB, 16 workers, 1 CTA)
# with the current kernel; C1 item size for tiny syncs
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
one() {  # label cfg
  timeout 600 python bench.py --config $2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-nv-supplied 2>/tmp/err.txt | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('$1 $2', d['value'], d['ms_min'], d['roofline']['frac'], d['clocks']['reasons'])" || tail -3 /tmp/err.txt
}
for v in 7 8 6; do for cfg in c10 c7 c11; do LLRL_CAST_VARIANT=$v one "v=$v" $cfg; done; done
for c in 8192 16384 4096; do
  LLRL_CHUNK_ELEMS=$c timeout 300 python bench.py --config c1 --steps 60 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > /tmp/o.json
  python -c "import json;d=json.loads(open('/tmp/o.json').read());print('c1 chunk=$c', d['value'], d['ms_min'], d.get('event_floor_us'))"
done
