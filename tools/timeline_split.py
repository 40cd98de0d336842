"""Per-CTA timeline of the split-K route kernel (debug).
usage: n d gathered [live]   (live: row count in device memory, n = capacity)"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
gathered = len(sys.argv) > 3 and sys.argv[3] == "1"
live = int(sys.argv[4]) if len(sys.argv) > 4 else None
n_dev = torch.tensor([live], dtype=torch.int64, device="cuda") if live is not None else None
b = 128
rows = 2 * n if gathered else n
h = torch.randn((rows, d), device="cuda").to(torch.bfloat16)
wd = (torch.randn((b, d), device="cuda") * 0.02).to(torch.bfloat16)
wu = torch.randn((b,), device="cuda") * 0.1
idx = torch.arange(0, rows, 2, device="cuda", dtype=torch.int64) if gathered else None
logits = torch.empty(n, device="cuda")
cont = torch.empty(n, dtype=torch.int64, device="cuda")
counts = torch.empty(2, dtype=torch.int64, device="cuda")
lib = N.load()
lib.tide_debug_timeline.argtypes = [ctypes.c_void_p]
dbg = torch.zeros(148 * 24, dtype=torch.int64, device="cuda")
ws = D.workspace().data_ptr()


def launch():
    N.check(lib.tide_route(h.data_ptr(), d, n, n_dev.data_ptr() if live is not None else None, rows, d, N.BF16,
                           idx.data_ptr() if gathered else None, wd.data_ptr(), wu.data_ptr(), b,
                           1e-6, 0.5, 3, None, logits.data_ptr(), None, None, cont.data_ptr(), 1,
                           None, counts.data_ptr(), ws, D.stream_handle()), "route")


for it in range(5):
    lib.tide_debug_timeline(dbg.data_ptr() if it == 4 else None)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    launch()
    e.record()
    torch.cuda.synchronize()
lib.tide_debug_timeline(None)
print(f"n={n} live={live} d={d} gathered={gathered}: event time of the traced launch {a.elapsed_time(e) * 1e3:.1f} us")
t = dbg.view(148, 24).cpu().numpy().astype(np.int64)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 0].min()
names = {0: "entry", 1: "setup_done", 2: "producer_issued", 3: "rms_done", 4: "acc_full",
         5: "pushed", 6: "cluster_sync1", 10: "logit_partials", 11: "finished_rows",
         8: "lookback_done", 7: "cluster_sync2", 9: "end"}
print(f"{t.shape[0]} CTAs; us relative to first CTA entry: min / median / max")
for k, nm in names.items():
    v = t[:, k]
    v = v[v > 0]
    if len(v):
        r = (v - t0) / 1000.0
        print(f"  {nm:16s} {r.min():8.2f} {np.median(r):8.2f} {r.max():8.2f}")
