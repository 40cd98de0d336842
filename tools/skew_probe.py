"""Is the per-SM streaming skew of K1 stable across launches?  Captures the
per-CTA timeline of several consecutive launches and correlates each SM's
finish time between them (profiling build: TIDE_PROBE_LIB=tools/_libs/*prof.so)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402
from paper_2603_21365_b200 import _native as N  # noqa: E402

lib = N.load(os.environ["TIDE_PROBE_LIB"]) if os.environ.get("TIDE_PROBE_LIB") else N.load()
lib.tide_debug_timeline.argtypes = [ctypes.c_void_p]
n, d, b = 65536, 4096, 128
g = torch.Generator(device="cuda")
g.manual_seed(0)
h = torch.randn((n, d), generator=g, device="cuda").to(torch.bfloat16)
wd = np.random.default_rng(1).standard_normal((b, d)).astype(np.float32) * 0.05
wu = np.random.default_rng(2).standard_normal((1, b)).astype(np.float32) * 0.1
router = P.Router(3, wd, wu)
runs = []
maps = []
for it in range(12):
    dbg = torch.zeros(148 * 24, dtype=torch.int64, device="cuda")
    lib.tide_debug_timeline(dbg.data_ptr() if it >= 4 else None)
    P.route(h, router, theta=0.5, want_indices=True, want_mask=True)
    torch.cuda.synchronize()
    if it >= 4:
        t = dbg.view(148, 24).cpu().numpy().astype(np.int64)
        fin = {int(t[i, 7]): (t[i, 1] - t[:, 0].min()) / 1e3 for i in range(148)}
        runs.append(fin)
        maps.append(tuple(int(x) for x in t[:, 7]))
lib.tide_debug_timeline(None)
sms = sorted(runs[0])
M = np.array([[r[s] for s in sms] for r in runs])
print("blockIdx->smid mapping identical across launches:", all(m == maps[0] for m in maps))
print("per-launch finish spread (us):", [round(float(x), 1) for x in (M.max(1) - M.min(1))])
C = np.corrcoef(M)
print("mean corr of per-SM finish time between launches: %.2f" % C[np.triu_indices(len(runs), 1)].mean())
dev = M - M.mean(1, keepdims=True)
print("per-SM mean deviation, slowest 8:", sorted(zip(dev.mean(0).round(2), sms))[-8:])
