# LM head TMA-store epilogue: parity tests, then A/B timing (interleaved rounds)
timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python - <<'PY'
import os, sys, json
sys.path.insert(0, '.')
import torch, bench_extra as B
for r in range(3):
    for st in ("0", "1"):
        for pair in ("1", "0"):
            os.environ["TIDE_LM_TMA_STORE"] = st
            os.environ["TIDE_LM_PAIR"] = pair
            x = B.lm_head()
            print(f"round {r} tma_store={st} pair={pair} 3term {x['ms_3term']:.3f} ms ({x['tflops_3term_bf16_mma']:.0f} TF/s) 1term {x['ms_1term_bf16']:.3f} ms ({x['tflops_1term']:.0f})", flush=True)
PY
