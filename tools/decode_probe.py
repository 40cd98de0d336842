"""Device time of the decode-step kernel (all checkpoints, one launch), CUDA-graph timed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402

for n in (1, 8, 16):
    for dt in (torch.bfloat16, torch.float32):
        ckpts, states, bank = BE._case(36, 4096, n, dt, 3, 0.3)
        cfg = P.RuntimeConfig(exit_threshold=0.5)
        gms = BE._graph_time(lambda: P.select_exits(states, bank, cfg), reps=20, inner=20)
        el = 2 if dt == torch.bfloat16 else 4
        byts = len(ckpts) * (n * 4096 * el + 128 * 4096 * el)
        print(f"n={n:2d} {str(dt):15s} {gms * 1e3:6.1f} us/step  {byts / (gms / 1e3) / 1e9:6.0f} GB/s", flush=True)
