timeout 120 python tools/chain_timeline.py 2>&1 | head -140
TIDE_CHAIN_FLAGS=1 timeout 120 python tools/chain_kernel_probe.py 2>&1 | tail -13
