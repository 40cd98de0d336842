timeout 600 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_posthoc.py -q -p no:cacheprovider --tb=short 2>&1 | tail -5
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_lmhead.py -q -p no:cacheprovider -k "tma_store and (129-256-129 or 2-128-4099)" 2>&1 | tail -8
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_lmhead.py -q -p no:cacheprovider -k "tma_store and 129-256-129" 2>&1 | tail -8
