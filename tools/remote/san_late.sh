mkdir -p gpurun_out/san
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 30 python tools/sanitize_cases.py late > gpurun_out/san/${tool}_late.log 2>&1
  echo "$tool late rc=$?"; grep -E "SUMMARY|sanitize cases ok" gpurun_out/san/${tool}_late.log | tail -2
done
