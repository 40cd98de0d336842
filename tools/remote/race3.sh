mkdir -p gpurun_out/san
timeout 900 python -m pytest tests/test_gpu_route.py tests/test_gpu_posthoc.py -q -p no:cacheprovider -x 2>&1 | tail -1
timeout 300 python tools/stress_k1.py 60 160000x2048 94720x128 2>&1 | grep reps
STRESS_F32=1 timeout 300 python tools/stress_k1.py 30 160000x1024 2>&1 | grep reps
SANITIZE_NO_DECODE=1 timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py k1m > gpurun_out/san/racecheck_k1m.log 2>&1; echo "racecheck k1m rc=$?"; tail -2 gpurun_out/san/racecheck_k1m.log
SANITIZE_NO_DECODE=1 timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py round1 > gpurun_out/san/racecheck_round1.log 2>&1; echo "racecheck round1 rc=$?"; tail -2 gpurun_out/san/racecheck_round1.log
