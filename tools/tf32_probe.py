"""f32 router launch (3xTF32 tensor-core kernel, or the CUDA-core kernel with
TIDE_F32_TC=0): device time per launch and logit error against an f64 torch
reference, |t - t64| / max(|t64|, m) with m = sum_j |w_up_j silu(a_j)|.
With TIDE_PROBE_LIB2=<lib>, also checks that lib gives bit-identical logits
(the TIDE_TF32_INPLACE=0 build: does the tensor core ignore the 13 low bits?)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402

lib = N.load(os.environ["TIDE_PROBE_LIB"]) if os.environ.get("TIDE_PROBE_LIB") else N.load()
lib2 = N.load(os.environ["TIDE_PROBE_LIB2"]) if os.environ.get("TIDE_PROBE_LIB2") else None
ws = D.workspace().data_ptr()
s = torch.cuda.current_stream().cuda_stream
shapes = [(2048, 768), (8192, 768), (1000, 772), (4096, 4096), (65536, 4096)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for shp in shapes:
    n, d = shp[:2]
    b = shp[2] if len(shp) > 2 else 128
    g = torch.Generator(device="cuda")
    g.manual_seed(n + d)
    h = torch.randn((n, d), generator=g, device="cuda") * 3.0
    wd = torch.randn((b, d), generator=g, device="cuda") * 0.05
    wu = torch.randn((b,), generator=g, device="cuda") * 0.3
    logits = torch.empty(n, device="cuda")
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    ei = torch.empty(n, dtype=torch.int64, device="cuda")
    ci = torch.empty(n, dtype=torch.int64, device="cuda")
    counts = torch.empty(2, dtype=torch.int64, device="cuda")

    def launch(L=lib, out=logits):
        N.check(L.tide_route(h.data_ptr(), d, n, None, n, d, N.F32, None, wd.data_ptr(),
                             wu.data_ptr(), b, 1e-6, 0.5, 3, None, out.data_ptr(),
                             mask.data_ptr(), ei.data_ptr(), ci.data_ptr(), 0, None,
                             counts.data_ptr(), ws, s), "route")

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    x = h.double()
    sc = 1.0 / torch.sqrt((x * x).sum(1) / d + 1e-6)
    a = (x @ wd.double().T) * sc[:, None]
    sl = a * torch.sigmoid(a)
    t64 = sl @ wu.double()
    m = (sl * wu.double()).abs().sum(1)
    err = ((logits.double() - t64).abs() / torch.maximum(t64.abs(), m)).max().item()
    line = (f"n={n:6d} d={d:5d} b={b:3d}  {us:8.1f} us  {n * d * 4 / us / 1e3:7.0f} GB/s  "
            f"max|dt|/max(|t|,m) = {err:.2e}  exits={int(counts[0])}")
    if lib2 is not None:
        l2 = torch.empty_like(logits)
        launch(lib2, l2)
        torch.cuda.synchronize()
        line += f"  bit-identical vs lib2: {bool(torch.equal(l2, logits))}"
    print(line, flush=True)
