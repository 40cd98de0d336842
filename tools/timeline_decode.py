"""Per-CTA timeline of the decode kernel (debug)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_extra as BE  # noqa: E402
import paper_2603_21365_b200 as P  # noqa: E402
from paper_2603_21365_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ckpts, states, bank = BE._case(36, 4096, n, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
lib = N.load()
lib.tide_debug_timeline.argtypes = [ctypes.c_void_p]
dbg = torch.zeros(148 * 24, dtype=torch.int64, device="cuda")
for it in range(6):
    lib.tide_debug_timeline(dbg.data_ptr() if it == 5 else None)
    P.select_exits(states, bank, cfg)
    torch.cuda.synchronize()
lib.tide_debug_timeline(None)
t = dbg.view(148, 24).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["entry", "loaded", "computed", "ticketed", "reduced(last)", "logit(last)", "resolved"]
print(f"{t.shape[0]} CTAs; us rel. to first entry: min / median / max (n>0 entries)")
for k, nm in enumerate(names):
    v = t[:, k]
    v = v[v > 0]
    if len(v):
        r = (v - t0) / 1000.0
        print(f"  {nm:14s} {r.min():7.2f} {np.median(r):7.2f} {r.max():7.2f}  ({len(v)})")
