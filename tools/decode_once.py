"""A few eager decode steps (config 3 shape) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402

ckpts, states, bank = BE._case(36, 4096, 8, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    P.select_exits(states, bank, cfg)
torch.cuda.synchronize()
print("ok")
