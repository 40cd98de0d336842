"""Kernel time via per-launch events vs back-to-back vs CUDA graph (same inputs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _native as N, _device as Dv
from oracle import tide_oracle as O
n, d, b = 65536, 4096, 128
g = np.random.Generator(np.random.PCG64(202))
orr = O.make_router(d, b, 3, g)
router = P.Router(3, orr.w_down, orr.w_up)
h = torch.randn((n, d), device="cuda").to(torch.bfloat16)
wd, wu = P.router_ops.device_weights(router, N.BF16, h.device)
sc = torch.empty(n, device="cuda"); mk = torch.empty(n, dtype=torch.uint8, device="cuda")
ex = torch.empty(n, dtype=torch.int64, device="cuda"); co = torch.empty_like(ex)
cnt = torch.empty(2, dtype=torch.int64, device="cuda")
lib = N.load(); ws = Dv.workspace().data_ptr()
def launch():
    s = torch.cuda.current_stream().cuda_stream
    lib.tide_route(h.data_ptr(), d, n, None, n, d, N.BF16, None, wd.data_ptr(), wu.data_ptr(), b, 1e-6, 0.5, 3,
                   sc.data_ptr(), None, mk.data_ptr(), ex.data_ptr(), co.data_ptr(), 0, None, cnt.data_ptr(), ws, s)
for _ in range(5): launch()
torch.cuda.synchronize()
# host cost per call
t0 = time.perf_counter()
for _ in range(200): launch()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host submit cost per call: {(t1 - t0) / 200 * 1e6:.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): launch()
e1.record(); torch.cuda.synchronize()
print(f"back-to-back: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per launch")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    launch()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20): launch()
    gr.replay(); torch.cuda.synchronize()
    e0.record(s)
    for _ in range(5): gr.replay()
    e1.record(s); torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us per launch")
