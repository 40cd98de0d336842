timeout 600 python -m pytest tests/test_gpu_posthoc.py -q -p no:cacheprovider -k "decode or config3" 2>&1 | tail -3
timeout 300 python - <<'PY'
import json, sys
sys.path.insert(0, '.')
import torch, bench_extra as B, paper_2603_21365_b200 as P
for args in [(), (P.BATCH_UNANIMOUS,), (P.PER_TOKEN, torch.float16)]:
    r = B.config3(*args); print(json.dumps({k: r[k] for k in ("config", "us_per_step_api", "us_per_step_graph", "gbs_graph")}))
PY
