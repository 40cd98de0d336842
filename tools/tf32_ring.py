"""3xTF32 route (f32 rows on tcgen05): device time per launch for ring shapes
TIDE_TF32_RING="nw,na,nl" (W slots, A slots, lo slots), logits / masks /
indices checked bit-identical against the default shape.
    python tools/tf32_ring.py 65536x4096 16384x8192x256 ...   (n x d [x b])"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402

lib = N.load()
ws = D.workspace().data_ptr()
s = torch.cuda.current_stream().cuda_stream
VARIANTS = [("default", {})] + [(f"ring {r}", {"TIDE_TF32_RING": r})
                               for r in os.environ.get("RINGS", "4,0,0 3,4,3 3,5,2 2,6,3 2,5,4").split()]
shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or [(65536, 4096)]
for shp in shapes:
    n, d = shp[:2]
    b = shp[2] if len(shp) > 2 else 128
    g = torch.Generator(device="cuda")
    g.manual_seed(n + d)
    h = torch.randn((n, d), generator=g, device="cuda") * 3.0
    wd = torch.randn((b, d), generator=g, device="cuda") * 0.05
    wu = torch.randn((b,), generator=g, device="cuda") * 0.3
    outs = {}
    for ring, env in VARIANTS:
        for k in ("TIDE_TF32_RING", "TIDE_TF32_PRESPLIT"):
            os.environ.pop(k, None)
        os.environ.update(env)
        logits = torch.empty(n, device="cuda")
        mask = torch.empty(n, dtype=torch.uint8, device="cuda")
        ei = torch.empty(n, dtype=torch.int64, device="cuda")
        ci = torch.empty(n, dtype=torch.int64, device="cuda")
        counts = torch.empty(2, dtype=torch.int64, device="cuda")

        def launch():
            N.check(lib.tide_route(h.data_ptr(), d, n, None, n, d, N.F32, None, wd.data_ptr(),
                                   wu.data_ptr(), b, 1e-6, 0.5, 3, None, logits.data_ptr(),
                                   mask.data_ptr(), ei.data_ptr(), ci.data_ptr(), 0, None,
                                   counts.data_ptr(), ws, s), "route")
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        best = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                launch()
            e1.record()
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1) / 10)
        ne = int(counts[0])
        res = (logits.clone(), mask.clone(), ei[:ne].clone(), ci[: n - ne].clone())
        if ring == "default":
            outs["ref"] = res
            same = True
        else:
            r0 = outs["ref"]
            same = all(torch.equal(a, b_) for a, b_ in zip(res, r0))
        ms = min(best)
        gbs = (n * d * 4 + b * d * 4) / (ms / 1e3) / 1e9
        print(f"{n}x{d} b={b} {ring}: {ms:.4f} ms  {gbs:.0f} GB/s  identical={same}", flush=True)
