TIDE_NVCC_EXTRA=-DTIDE_DECODE_DEBUG python -m paper_2603_21365_b200.build --force > /dev/null 2>&1
TIDE_PDL=0 TIDE_ALLOW_STALE=1 timeout 120 python tools/decode_once.py 1 2>&1 | grep "send\|hang\|blk1" | sort | head -70
