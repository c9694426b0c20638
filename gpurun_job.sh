cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python tools/sweep.py --out gpurun_out/sweep_fp32.jsonl > gpurun_out/sweep_fp32.md 2>&1
timeout 900 python tools/sweep.py --dq --min-log2 24 --out gpurun_out/sweep_dq.jsonl > gpurun_out/sweep_dq.md 2>&1
for cfg in cfg1 cfg3; do timeout 900 python bench.py --config $cfg --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; done
timeout 900 python bench.py --config cfg4 --scaling strong --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_rank0of8.json 2>gpurun_out/bench_cfg4.err
tail -3 gpurun_out/sweep_fp32.md; for f in gpurun_out/bench_cfg*.json; do python -c "import json;d=json.load(open('$f'));print('$f', d['value'], d['roofline']['frac'], d['config']['elements_per_rank'])"; done
