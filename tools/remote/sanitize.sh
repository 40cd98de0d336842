mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san/$tool.log
done
