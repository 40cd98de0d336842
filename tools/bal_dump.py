"""Dump the adaptive-balance table of the route kernel's workspace after a few launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402

lib = N.load(os.environ["TIDE_PROBE_LIB"]) if os.environ.get("TIDE_PROBE_LIB") else N.load()
n, d, b = 65536, 4096, 128
g = torch.Generator(device="cuda")
g.manual_seed(0)
h = torch.randn((n, d), generator=g, device="cuda").to(torch.bfloat16)
wd = np.random.default_rng(1).standard_normal((b, d)).astype(np.float32) * 0.05
wu = np.random.default_rng(2).standard_normal((1, b)).astype(np.float32) * 0.1
router = P.Router(3, wd, wu)
ws = D.workspace()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    P.route(h, router, theta=0.5, want_indices=True, want_mask=True)
    torch.cuda.synchronize()
    w = ws[:4 * (8 + 4 * 256)].view(torch.int32).cpu().numpy()
    par = (w[0] & 1) ^ 1  # buffer written by the launch that just ran
    bw = w[8 + par * 256: 8 + par * 256 + 148]
    bt = w[8 + 512 + par * 256: 8 + 512 + par * 256 + 148] / 1e3
    print("epoch %d  w min/max %d/%d  t min/mean/max %.1f/%.1f/%.1f us" % (w[0], bw.min(), bw.max(), bt.min(), bt.mean(), bt.max()))
