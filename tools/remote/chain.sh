timeout 300 python -m pytest tests/test_gpu_chain.py -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 600 python bench_extra.py sweep 2>&1 | tail -8
