timeout 900 python -m pytest tests/test_gpu_route.py -q -x -p no:cacheprovider --tb=short -k "f32" 2>&1 | tail -5
timeout 600 python tools/tf32_ring.py 65536x4096 65536x4096x64 65536x4096x96 65536x4096x160 65536x4096x256 16384x8192 65536x768 4096x4096 2>&1 | tail -40
