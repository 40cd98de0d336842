timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 300 python bench_extra.py lm 2>&1 | tail -3
