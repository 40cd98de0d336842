# LM head persistent CTA pairs: parity tests, then A/B timing (interleaved rounds)
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_posthoc.py -q -x -p no:cacheprovider --tb=short 2>&1 | tail -15
timeout 600 python - <<'PY'
import os, sys, json
sys.path.insert(0, '.')
import torch, bench_extra as B
os.environ["TIDE_LM_PAIR"] = "1"
for r in range(3):
    for per in ("0", "1"):
        os.environ["TIDE_LM_PERSIST"] = per
        x = B.lm_head()
        print(f"round {r} persist={per} 3term {x['ms_3term']:.3f} ms ({x['tflops_3term_bf16_mma']:.0f} TF/s) 1term {x['ms_1term_bf16']:.3f} ms ({x['tflops_1term']:.0f})", flush=True)
PY
