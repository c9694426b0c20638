cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -4
timeout 300 python tools/gemm_probe.py 16 4096 5376
timeout 300 python tools/gemm_probe.py 16 21504 5376
timeout 300 python tools/gemm_probe.py 128 21504 5376
for m in 1 16 64 256; do timeout 300 python tools/gemm_bench.py --m $m --layers 8 --steps 10 2>&1 | tail -1; done
