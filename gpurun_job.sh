cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b_f4.json 2> gpurun_out/b_f4.err
python -c "import json;d=json.load(open('gpurun_out/b_f4.json'));print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d.get('sol_stream_gbs'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/b_f4.err
