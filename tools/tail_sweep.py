"""Configs 2 and 5 (graph-timed) under tail settings from the environment:
TIDE_TAIL_AFTER (links before the tail), TIDE_TAIL_ROWS (row limit at d=4096),
TIDE_TAIL_KS (tail cluster-size cap)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as B  # noqa: E402

tag = " ".join(f"{k}={os.environ[k]}" for k in ("TIDE_TAIL_AFTER", "TIDE_TAIL_ROWS", "TIDE_TAIL_KS")
               if k in os.environ)
for fn in (B.config2, B.config5):
    r = fn()
    print(json.dumps({"tag": tag, "config": r["config"][:2], "ms_graph": round(r["ms_graph"], 4)}),
          flush=True)
