RINGS="2,0,0" timeout 600 python tools/tf32_ring.py 65536x4096 32768x4096 16384x8192 65536x768 2>&1 | tail -8
TIDE_F32_TC=1 RINGS="2,0,0" timeout 600 python tools/tf32_ring.py 4096x4096 8192x2048 2>&1 | tail -4
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -8
