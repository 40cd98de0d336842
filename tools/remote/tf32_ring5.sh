RINGS="2,4,4 2,5,4 2,4,3 3,4,3 3,4,2 4,4,1" timeout 600 python tools/tf32_ring.py 65536x4096 16384x8192 65536x1024 2>&1 | tail -21
