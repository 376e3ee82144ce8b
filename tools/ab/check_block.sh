# 1 GPU: parity of the block default for quantising plans + their table lines
cd $GRAFT_REPO_ROOT
rev=$(cat .git_rev)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -q -k "toy or edge or guard or long_items" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvfp4.py -m gpu -q -k "full and (c7 or c10 or c11 or c12)" 2>&1 | tail -2
echo "($rev)"
bash tools/gpu.sh table 1 c7 c10 c11 c12 c2
