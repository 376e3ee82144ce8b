# 1 GPU at the last code commit: the whole GPU suite + smoke + the default bench line
cd $GRAFT_REPO_ROOT
rev=$(cat .git_rev)
bash tools/gpu.sh tests
sed -i "s/(snapshot)/($rev)/" gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final_bench_n1_last.json 2> gpurun_out/final_bench_n1_last.err
tail -c 400 gpurun_out/final_bench_n1_last.json
