python tools/timeline_decode_graph.py 8 10 2>&1 | head -40
python - <<'PY'
import json, sys
sys.path.insert(0, '.')
import torch, bench_extra as B, paper_2603_21365_b200 as P
for args in [(), (P.BATCH_UNANIMOUS,), (P.PER_TOKEN, torch.float16)]:
    r = B.config3(*args); print(json.dumps({k: r[k] for k in ("us_per_step_api", "us_per_step_graph")}))
PY
