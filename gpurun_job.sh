cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in v2u4 v2u4s v2u4sx v2u4sxc v2u4c v2u4xc; do
  timeout 600 python bench.py --steps 50 --warmup 5 --variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench_var_$v.json 2> gpurun_out/bench_var_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_var_$v.json'));print('$v', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d.get('sol_stream_gbs'), d['clocks'])" || tail -3 gpurun_out/bench_var_$v.err
done
