cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nf4_gemm_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_v7 python tools/gemm_prof_case.py > /dev/null 2>&1
