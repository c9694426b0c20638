cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
timeout 300 python tools/gemm_probe.py 16 4096 5376
timeout 300 python tools/gemm_probe.py 16 21504 5376
python -c "
import paper_2604_02556_b200 as n
for (M,N,K) in [(16,4096,5376),(16,21504,5376),(16,5376,21504),(128,21504,5376),(1,2048,5376)]: print(M,N,K,n.nf4_gemm_default_splits(M,N,K))"
for m in 1 16 64; do timeout 300 python tools/gemm_bench.py --m $m --layers 8 --steps 10 2>&1 | tail -1; done
