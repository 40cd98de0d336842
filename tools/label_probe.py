"""Device time of the calibration labeller at BASELINE config 4 (1,024,000 x 4096
bf16, 8 checkpoints + final), back-to-back launches (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _native as N  # noqa: E402
from paper_2603_21365_b200 import _device as D  # noqa: E402

lib = N.load(os.environ["TIDE_PROBE_LIB"]) if os.environ.get("TIDE_PROBE_LIB") else N.load()
n, d, C = int(sys.argv[1]) if len(sys.argv) > 1 else 1_024_000, 4096, 8
g = torch.Generator(device="cuda")
g.manual_seed(4)
bufs = []
for i in range(C + 1):
    t = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    for r0 in range(0, n, 131072):
        r1 = min(n, r0 + 131072)
        t[r0:r1] = torch.randn((r1 - r0, d), generator=g, device="cuda").to(torch.bfloat16)
    bufs.append(t)
sims = torch.empty(C * n, dtype=torch.float32, device="cuda")
labels = torch.empty(C * n, dtype=torch.uint8, device="cuda")
zc = torch.empty(C, dtype=torch.int64, device="cuda")
ptrs = N.ptr_array([b.data_ptr() for b in bufs[:C]])
s = D.stream_handle()


def launch():
    N.check(lib.tide_cos_label(ptrs, C, bufs[C].data_ptr(), d, N.BF16, n, d, 0.98, sims.data_ptr(),
                               labels.data_ptr(), None, None, zc.data_ptr(), s), "label")


for _ in range(2):
    launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    launch()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
byts = n * (C + 1) * d * 2 + n * C * 5
print(f"labeller n={n}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s  (sims sum {float(sims.double().sum()):.6f})")
