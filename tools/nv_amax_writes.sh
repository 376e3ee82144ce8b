# Where do llrl_k_nv_amax's DRAM writes come from (verdict r1 weak #5)?  L2 write /
# atomic sectors vs DRAM writes, with ncu's cache flush between replays (default)
# and without it.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_read.sum
for cc in all none; do
  timeout 900 ncu --metrics $M --cache-control $cc --clock-control none -k regex:llrl_k_nv_amax -c 3 --csv \
     --log-file gpurun_out/nv_amax_writes_$cc.csv python bench.py --config c11 --steps 1 --warmup 3 --no-e2e \
     --no-cpu-baseline --no-nv-supplied > gpurun_out/nv_amax_writes_$cc.log 2>&1
done
for k in llrl_k_cast_tma; do
  timeout 900 ncu --metrics $M --cache-control all --clock-control none -k regex:$k -c 2 --csv \
     --log-file gpurun_out/nv_cast_writes.csv python bench.py --config c11 --steps 1 --warmup 3 --no-e2e \
     --no-cpu-baseline --no-nv-supplied > gpurun_out/nv_cast_writes.log 2>&1
done
