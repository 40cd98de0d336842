timeout 600 python -m pytest tests/test_hook.py tests/test_gpu_advice_r01.py -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 900 python tools/hook_bench.py 20 2>&1 | tail -5
