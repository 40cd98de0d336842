mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py k1m > gpurun_out/san/racecheck_k1m.log 2>&1; echo "racecheck k1m rc=$?"; tail -2 gpurun_out/san/racecheck_k1m.log
timeout 1700 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py round1 > gpurun_out/san/racecheck_round1.log 2>&1; echo "racecheck round1 rc=$?"; tail -2 gpurun_out/san/racecheck_round1.log
