"""Per-CTA timeline of the tensor-core route kernel (debug): where does time go?"""
import ctypes, json, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _native as N, _device as Dv
from oracle import tide_oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
d, b = 4096, 128
g = np.random.Generator(np.random.PCG64(202))
orr = O.make_router(d, b, 3, g)
router = P.Router(3, orr.w_down, orr.w_up)
h = torch.randn((n, d), device="cuda").to(torch.bfloat16)
lib = N.load(os.environ['TIDE_PROBE_LIB']) if os.environ.get('TIDE_PROBE_LIB') else N.load()
lib.tide_debug_timeline.argtypes = [ctypes.c_void_p]
dbg = torch.zeros(148 * 24, dtype=torch.int64, device="cuda")
for it in range(4):
    lib.tide_debug_timeline(dbg.data_ptr() if it == 3 else None)
    P.route(h, router, theta=0.5, want_indices=os.environ.get('TL_NOSCAN') != '1', want_mask=True)
torch.cuda.synchronize()
lib.tide_debug_timeline(None)
t = dbg.view(148, 24).cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
cols = [0, 1, 2, 8, 9, 10, 11, 12, 13, 14, 15, 3, 4, 5, 6]
rel = (t[:, cols] - t0) / 1000.0
names = ["start", "prod_done", "stream_done", "tfull0", "tile0_done", "tfull1", "tile1_done", "tfull2", "tile2_done", "tfull3", "tile3_done", "epi_done", "scan_start", "lookback_done", "end"]
print("us rel. to first CTA start: min / median / max per event")
for i, nm in enumerate(names):
    if np.all(t[:, cols[i]] == 0): continue
    print(f"{nm:14s} {rel[:, i].min():8.1f} {np.median(rel[:, i]):8.1f} {rel[:, i].max():8.1f}")
np.save("gpurun_out/timeline.npy", t)

c = t[:, 16:22].astype(np.float64)
c = c[(c[:, 1] > 0)]
print("MMA thread: wait %.0f%% of %.0f cyc | producer: wait %.0f%% of %.0f cyc | rms warp: wait %.0f%% of %.0f cyc" % (
    100 * np.median(c[:, 0] / c[:, 1]), np.median(c[:, 1]), 100 * np.median(c[:, 2] / c[:, 3]), np.median(c[:, 3]),
    100 * np.median(c[:, 4] / c[:, 5]), np.median(c[:, 5])))
