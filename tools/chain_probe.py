"""Launch list of one per-token posthoc chain (BASELINE config 2 or 5) for ncu:
    ncu --metrics gpu__time_duration.sum --clock-control none python tools/chain_probe.py 2"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as B  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402

cfgn = sys.argv[1] if len(sys.argv) > 1 else "2"
if cfgn == "2":
    ckpts, states, bank = B._case(32, 4096, 4096, torch.bfloat16, 2, 0.1)
    cfg = P.RuntimeConfig(exit_threshold=0.5)
else:  # bench_extra.config5's case
    ckpts, states, bank = B._case(80, 8192, 8192, torch.bfloat16, 5, 0.06)
    cfg = P.RuntimeConfig(exit_threshold=0.7)
for _ in range(3):
    exits = P.select_exits(states, bank, cfg)
torch.cuda.synchronize()
e = exits.cpu()
rem = len(e)
for k in ckpts:
    print(f"ckpt {k}: rows in {rem}, exit {(e == k).sum().item()}")
    rem -= (e == k).sum().item()
