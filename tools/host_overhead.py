"""Host-side cost of one decode-step select_exits call (cProfile + wall time)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402

ckpts, states, bank = BE._case(36, 4096, 8, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
for _ in range(50):
    P.select_exits(states, bank, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    P.select_exits(states, bank, cfg)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host time per call: {(t1 - t0) / 2000 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    P.select_exits(states, bank, cfg)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

step = P.DecodeStep(states, bank, cfg)
for _ in range(50):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"DecodeStep host time per call: {(t1 - t0) / 2000 * 1e6:.1f} us")
