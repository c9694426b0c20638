cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "beyond" 2>&1 | tail -2
