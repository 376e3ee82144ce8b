# does test_long_items_claimed_phase catch the by-reference hand-off bug? (HEAD must pass, _ab/byref must fail)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _ab/byref && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
echo "== HEAD"; timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "long_items" 2>&1 | tail -3
echo "== byref"; (cd _ab/byref && timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "long_items" 2>&1 | tail -6)
