"""Decode-step time per graph replay, 5 samples (timing experiments: swap tools/_libs/dec*.so in)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench_extra as BE
import paper_2603_21365_b200 as P
ckpts, states, bank = BE._case(36, 4096, 8, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
vals = [BE._graph_time(lambda: P.select_exits(states, bank, cfg), reps=20, inner=20) * 1e3 for _ in range(5)]
print(sys.argv[1], " ".join(f"{v:.2f}" for v in vals), "us/step")
