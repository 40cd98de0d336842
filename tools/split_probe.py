"""Per-launch device time of K1 (split-K cluster vs persistent) over row counts."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P  # noqa: E402
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402


def run(n, d, b=128, reps=20, gathered=False):
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    rows = n * 2 if gathered else n
    h = torch.randn((rows, d), generator=g, device="cuda").to(torch.bfloat16)
    wd = (torch.randn((b, d), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    wu = torch.randn((b,), generator=g, device="cuda") * 0.1
    idx = torch.arange(0, rows, 2, device="cuda", dtype=torch.int64) if gathered else None
    logits = torch.empty(n, device="cuda")
    counts = torch.empty(2, dtype=torch.int64, device="cuda")
    cont = torch.empty(n, dtype=torch.int64, device="cuda")
    lib = N.load()
    ws = D.workspace().data_ptr()
    s = None

    def launch():
        N.check(lib.tide_route(h.data_ptr(), d, n, None, rows, d, N.BF16,
                               idx.data_ptr() if gathered else None, wd.data_ptr(), wu.data_ptr(),
                               b, 1e-6, 0.5, 3, None, logits.data_ptr(), None, None,
                               cont.data_ptr(), 1, None, counts.data_ptr(), ws, s), "route")
    # device time: reps launches captured in one CUDA graph (no host gaps)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        s = D.stream_handle()
        launch()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(reps):
                launch()
        gr.replay()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        gr.replay()
        e.record(st)
        torch.cuda.synchronize()
    return a.elapsed_time(e) / reps * 1e3


for d in (4096, 8192):
    for n in (128, 512, 1024, 2048, 4096, 8192, 16384):
        for gathered in (False, True):
            res = {}
            for mode in ("8", "4", "2", "0"):
                os.environ["TIDE_SPLIT"] = mode
                res[mode] = run(n, d, gathered=gathered)
            byts = n * d * 2
            print(f"d={d} n={n:6d} g={int(gathered)} " + "  ".join(
                f"ks<={m}: {v:6.1f} us {byts / v / 1e3:5.0f} GB/s" for m, v in res.items()),
                flush=True)
