"""Device time of batch_compact with the row gather (exactly-sized exit /
continuing row outputs) at hidden-state widths: bytes moved = the rows read
once + written once.
    python tools/compact_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402

for n, d, dt in ((65536, 4096, torch.bfloat16), (16384, 4096, torch.bfloat16), (65536, 768, torch.float32),
                 (65536, 16, torch.float32)):
    h = torch.randn((n, d), device="cuda").to(dt)
    mask = torch.rand(n, device="cuda") < 0.5
    for _ in range(3):
        P.batch_compact(h, mask)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    R = 10
    for _ in range(R):
        P.batch_compact(h, mask)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / R
    byts = 2 * n * d * h.element_size()
    print(f"n={n} d={d} {dt}: {ms * 1e3:.1f} us per call (incl. host), {byts / ms / 1e6:.0f} GB/s moved", flush=True)
