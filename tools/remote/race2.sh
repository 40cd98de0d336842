mkdir -p gpurun_out/san
timeout 600 python -m pytest tests/test_gpu_posthoc.py -q -p no:cacheprovider -k "repeats_bitwise" 2>&1 | tail -1
SANITIZE_NO_DECODE=1 timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py k1m > gpurun_out/san/racecheck_k1m.log 2>&1; echo "racecheck k1m rc=$?"; tail -2 gpurun_out/san/racecheck_k1m.log
