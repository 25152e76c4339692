# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py -> gpurun_out/sanitize_*.txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sanitize_cases.py 2>&1 | tail -1
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 2000 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
echo done
