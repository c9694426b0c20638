cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for tool in initcheck; do
  echo "== $tool"
  NF4_SANITIZE_DEFAULT_ONLY=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
