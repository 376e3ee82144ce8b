cd $GRAFT_REPO_ROOT
bash tools/nv_amax_writes.sh
bash tools/gpu.sh ncufull c12 llrl_k_cast_tma
bash tools/gpu.sh ncufull c11 llrl_k_cast_tma
bash tools/gpu.sh ncufull c12 llrl_k_nv_amax
for f in gpurun_out/ncu_c1*_llrl_k_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}.raw.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep
