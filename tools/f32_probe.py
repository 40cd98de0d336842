"""Device time of the f32 router launch (route_simt) at config 1 and headline shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402
from oracle import tide_oracle as O  # noqa: E402

for n, d in ((2048, 768), (8192, 768), (4096, 4096), (65536, 4096)):
    g = np.random.Generator(np.random.PCG64(1))
    r = O.make_router(d, 128, 3, g)
    h = torch.randn((n, d), device="cuda")
    for dt in (torch.float32, torch.bfloat16):
        x = h.to(dt)
        ms = BE._time(lambda: P.fused_layernorm_route(x, r), reps=20)
        gms = BE._graph_time(lambda: P.fused_layernorm_route(x, r), reps=20)
        byts = n * d * x.element_size()
        print(f"n={n:6d} d={d:5d} {str(dt):15s} api {ms * 1e3:8.1f} us  graph {gms * 1e3:8.1f} us "
              f"{byts / (gms / 1e3) / 1e9:7.0f} GB/s  {2 * n * d * 128 / (gms / 1e3) / 1e12:6.1f} TFLOP/s",
              flush=True)
