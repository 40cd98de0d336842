"""Determinism stress of the LM head (persistent CTA pairs by default): one
launch repeated with an L2-thrashing fill in between, logits compared bitwise.
    python tools/stress_lm.py [reps] [n d V]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402
from paper_2603_21365_b200.runtime import split_bf16  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n, d, V = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (4096, 4096, 50257)
g = torch.Generator(device="cuda")
g.manual_seed(3)
a = torch.randn((n, d), generator=g, device="cuda")
w = torch.randn((V, d), generator=g, device="cuda") * 0.02
ld = (d + 7) // 8 * 8
ah, al = split_bf16(a, ld)
bh, bl = split_bf16(w, ld)
ldo = (V + 3) // 4 * 4
lib = N.load()
s = D.stream_handle(torch.device("cuda", 0))
junk = torch.empty(1 << 27, device="cuda")
bad = 0
for terms in (3, 1):
    ref = None
    for i in range(reps):
        out = torch.empty((n, ldo), device="cuda")
        N.check(lib.tide_lm_head(ah.data_ptr(), al.data_ptr() if terms == 3 else None, ld, n, d,
                                 bh.data_ptr(), bl.data_ptr() if terms == 3 else None, ld, V,
                                 out.data_ptr(), ldo, s), "lm_head")
        junk.fill_(float(i))
        if ref is None:
            ref = out[:, :V].clone()
        elif not torch.equal(out[:, :V], ref):
            bad += 1
    torch.cuda.synchronize()
    print(f"terms={terms} n={n} d={d} V={V} reps={reps} mismatches so far {bad}", flush=True)
print("MISMATCHES", bad)
