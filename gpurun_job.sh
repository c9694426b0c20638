cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/layer_latency.py --model gemma-3-27b 2>&1 | tail -1
timeout 900 python tools/sweep.py --max-log2 26 2>&1 | awk '/\| 64 \| bf16/'
