cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/gemm_probe.py 16 21504 5376
for m in 1 16 64; do timeout 300 python tools/gemm_bench.py --m $m --layers 8 --steps 10 --no-unfused 2>&1 | tail -1; done
timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"
