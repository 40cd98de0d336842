"""Per-CTA timeline of the decode kernel inside a CUDA graph of K steps
(steady state: W and the rows L2-resident, launches back to back).

    python tools/timeline_decode_graph.py [rows] [steps]

Slots are clock64 stamps (decode.cu DTL); printed in us at the measured SM
clock, relative to the step's first CTA entry; plus the launch gap between
steps from the entries' globaltimer."""
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
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ckpts, states, bank = BE._case(36, 4096, n, torch.bfloat16, 3, 0.3)
cfg = P.RuntimeConfig(exit_threshold=0.5)
lib = N.load()
lib.tide_debug_timeline.argtypes = [ctypes.c_void_p]
SL = 32


def run(with_tl):
    dbg = torch.zeros((K, 148 * SL), dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for k in range(K):
                lib.tide_debug_timeline(dbg[k].data_ptr() if with_tl else None)
                P.select_exits(states, bank, cfg)
        lib.tide_debug_timeline(None)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        dbg.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3, dbg


P.select_exits(states, bank, cfg)
torch.cuda.synchronize()
us0, _ = run(False)
us1, dbg = run(True)
print(f"graph of {K} steps: {us0:.2f} us/step ({us1:.2f} with the timeline)")
names = {12: "dep released", 0: "entry", 8: "W landed", 9: "MMAs issued", 1: "h landed", 2: "acc in smem",
         3: "recv ready", 7: "summed", 4: "logits", 5: "score", 6: "atomic done"}
T = dbg.view(K, 148, SL).cpu().numpy().astype(np.int64)
t = T[K - 1]
t = t[t[:, 31] > 0]
# clock rate from the two globaltimer-stamped ends is not available per slot:
# use the nominal measured clock of the box for conversion
mhz = float(os.environ.get("SM_MHZ", "1965"))
print(f"step {K - 1}: {t.shape[0]} CTAs; us (at {mhz:.0f} MHz) rel. to each CTA's entry: "
      "min / median / max")
for j in (0, 12, 1, 8, 9, 2, 3, 7, 4, 5, 6):
    ok = t[:, j] > 0
    if ok.any():
        r = (t[ok, j] - t[ok, 0]) / mhz
        print(f"  {names[j]:12s} {r.min():7.2f} {np.median(r):7.2f} {r.max():7.2f}  ({int(ok.sum())})")
e = t[:, 31]
print(f"entry skew across CTAs (globaltimer) us: {(e.max() - e.min()) / 1e3:.2f}")
starts = [T[k][T[k][:, 31] > 0][:, 31].min() for k in range(K)]
print(f"entry-to-entry (globaltimer) us: median {np.median(np.diff(starts)) / 1e3:.2f}")
