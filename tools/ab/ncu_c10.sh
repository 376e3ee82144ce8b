# ncu --set full of the C10 (MXFP4) cast kernel: HEAD vs a80a60a (where is the 5%?)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _ab/a80a60a && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
for t in head a80a60a; do
  d=.; [ $t = a80a60a ] && d=_ab/a80a60a
  (cd $d && timeout 900 ncu --set full --clock-control none --import-source on -k regex:llrl_k_cast_tma -c 1 \
      -o $GRAFT_REPO_ROOT/gpurun_out/ncu_c10_$t python bench.py --config c10 --steps 1 --warmup 3 --no-e2e \
      --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/ncu_c10_$t.log 2>&1)
  ncu -i gpurun_out/ncu_c10_$t.ncu-rep --page raw --csv > gpurun_out/ncu_c10_$t.raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu_c10_$t.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_c10_$t.sass.csv 2>/dev/null
done
ls -la gpurun_out/ncu_c10_*
