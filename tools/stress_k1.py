"""Determinism stress of K1 (route_tc): the same launch repeated must give
bit-identical logits / mask / indices / counts (fixed reduction orders), with
other kernels (a fresh fill of an unrelated buffer, a K1m chain) interleaved.
    python tools/stress_k1.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402
from oracle import tide_oracle as O  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
bad = 0
shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[2:]] or \
    [(160_000, 256), (65_536, 4096), (100_000, 256), (40_960, 1024)]
for n, d in shapes:
    bad_shape = 0
    g = np.random.Generator(np.random.PCG64(n + d))
    wd = (g.standard_normal((128, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, 128)) * 0.05).astype(np.float32)
    router = P.Router(layer=3, w_down=wd, w_up=wu)
    dt = torch.float32 if os.environ.get("STRESS_F32") == "1" else torch.bfloat16
    h = torch.randn((n, d), device="cuda").to(dt)
    junk = torch.empty(1 << 26, device="cuda")
    ref = P.route(h, router, theta=0.5, want_logits=True, want_indices=True)
    ref = {k: v.clone() for k, v in ref.items() if torch.is_tensor(v)}
    for i in range(reps):
        junk.fill_(float(i))
        r = P.route(h, router, theta=0.5, want_logits=True, want_indices=True)
        for k, v in ref.items():
            if r[k].shape != v.shape or not torch.equal(r[k], v):
                bad += 1
                bad_shape += 1
                if bad_shape <= 3 and r[k].shape == v.shape:
                    diff = (r[k] != v).nonzero().flatten()[:8].tolist()
                    print(f"n={n} d={d} rep {i}: {k} differs at {diff} ({int((r[k] != v).sum())} elements)")
    print(f"n={n} d={d}: {reps} reps, {bad_shape} mismatching outputs", flush=True)
print("MISMATCHES", bad)
