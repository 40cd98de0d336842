"""Device time of exit_projection / exit_scatter (rows read once, written once
into their positions) and select_project_split staging at hidden-state widths.
    python tools/project_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402


def t(fn, R=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(R):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / R


for n, d, dt in ((32768, 4096, torch.bfloat16), (32768, 4096, torch.float32), (8192, 768, torch.float32)):
    ex = torch.randn((n, d), device="cuda").to(dt)
    pos = torch.arange(0, 2 * n, 2, device="cuda", dtype=torch.int64)
    out = torch.empty((2 * n, d), device="cuda", dtype=torch.float32)
    gain = np.ones(d, np.float32)
    ms_p = t(lambda: P.exit_projection(ex, gain, 1e-6, pos, out))
    ms_s = t(lambda: P.exit_scatter(ex.float() if dt != torch.float32 else ex, pos, out))
    byts = n * d * (ex.element_size() + 4)
    print(f"n={n} d={d} {dt}: exit_projection {ms_p * 1e3:.1f} us ({byts / ms_p / 1e6:.0f} GB/s), "
          f"exit_scatter {ms_s * 1e3:.1f} us", flush=True)
