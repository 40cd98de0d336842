"""Host cost of one eager select_exits call on the config-2 chain (cProfile)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402

ckpts, states, bank = BE._case(32, 4096, 4096, torch.bfloat16, 2, 0.1)
cfg = P.RuntimeConfig(exit_threshold=0.5)
for _ in range(20):
    P.select_exits(states, bank, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    P.select_exits(states, bank, cfg)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue time per call: {(t1 - t0) / 200 * 1e6:.1f} us; with drain {(t2 - t0) / 200 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    P.select_exits(states, bank, cfg)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
