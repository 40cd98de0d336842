mkdir -p gpurun_out/san
for tool in memcheck synccheck initcheck racecheck; do
  for grp in round1 round2 k1m; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py $grp > gpurun_out/san/${tool}_${grp}.log 2>&1
    echo "$tool $grp rc=$?"; grep -E "SUMMARY|sanitize cases ok" gpurun_out/san/${tool}_${grp}.log | tail -2
  done
done
