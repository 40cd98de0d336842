timeout 900 python -m pytest tests/test_gpu_route.py tests/test_gpu_posthoc.py tests/test_gpu_pdl.py -q -p no:cacheprovider --tb=short -k "f32 or tf32 or pdl" 2>&1 | tail -5
timeout 600 python tools/tf32_ring.py 65536x4096 16384x4096 16384x8192 65536x768 8192x768 2>&1 | tail -16
