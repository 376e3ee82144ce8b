# 1 GPU: the strided-source amax-run rule -- parity (run lengths, full C11 / C12) and C11 / C12 lines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -q -k "nv_amax_runs or (nvfp4 and toy)" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "full_70b_every_byte and (c11 or c12)" 2>&1 | tail -2
echo "($(cat .git_rev))"
bash tools/gpu.sh table 1 c12 c11
