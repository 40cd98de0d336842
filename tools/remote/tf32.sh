for acc in 1 2 4; do echo "== TIDE_TF32_ACC=$acc"; TIDE_F32_TC=1 TIDE_TF32_ACC=$acc timeout 300 python tools/tf32_probe.py 2048x768 1000x772 4096x4096 65536x4096 8192x8192 2048x16384 2>&1 | tail -6; done
echo "== CUDA cores"; TIDE_F32_TC=0 timeout 300 python tools/tf32_probe.py 4096x4096 65536x4096 8192x8192 2>&1 | tail -3
