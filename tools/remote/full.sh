timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r2_gpu_tests.log | tail -5
bash tools/remote/sanitize.sh
