"""One select_exits call at config 2 or 5 (for ncu launch lists):
    python tools/chain_once.py <config 2|5> <theta> [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as B  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402

cfg_id, theta = sys.argv[1], float(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if cfg_id == "2":
    ckpts, states, bank = B._case(32, 4096, 4096, torch.bfloat16, 2, 0.1)
else:
    ckpts, states, bank = B._case(80, 8192, 8192, torch.bfloat16, 5, 0.06)
cfg = P.RuntimeConfig(exit_threshold=theta)
os.environ["TIDE_CHAIN_GRAPHS"] = "0"
for _ in range(reps):
    e = P.select_exits(states, bank, cfg)
torch.cuda.synchronize()
print("exit rate", float((e >= 0).float().mean()))
