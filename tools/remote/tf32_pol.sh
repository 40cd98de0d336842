S="1024x1024 4096x1024 16384x1024 65536x1024 1024x2048 4096x2048 16384x2048 1024x4096 2048x4096 4096x4096 8192x4096 1024x8192 4096x8192 8192x8192"
echo "== simt"; TIDE_F32_TC=0 timeout 300 python tools/tf32_probe.py $S 2>&1 | tail -14
echo "== tc presplit"; TIDE_F32_TC=1 timeout 300 python tools/tf32_probe.py $S 2>&1 | tail -14
echo "== tc in-kernel split"; TIDE_F32_TC=1 TIDE_TF32_PRESPLIT=0 timeout 300 python tools/tf32_probe.py $S 2>&1 | tail -14
