"""Run K1 at the headline shape back to back for a few seconds while sampling
nvidia-smi (power, SM clock, throttle reasons) — is the fused kernel power-capped?"""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402

n, d, b = 65536, 4096, 128
g = torch.Generator(device="cuda")
g.manual_seed(0)
zero = os.environ.get("PP_ZERO") == "1"
h = torch.zeros((n, d), device="cuda", dtype=torch.bfloat16) if zero else \
    torch.randn((n, d), generator=g, device="cuda").to(torch.bfloat16)
wd = (torch.randn((b, d), generator=g, device="cuda") * 0.05).to(torch.bfloat16)
wu = torch.randn((b,), generator=g, device="cuda") * 0.1
scores = torch.empty(n, device="cuda")
mask = torch.empty(n, dtype=torch.uint8, device="cuda")
ei = torch.empty(n, dtype=torch.int64, device="cuda")
ci = torch.empty(n, dtype=torch.int64, device="cuda")
counts = torch.empty(2, dtype=torch.int64, device="cuda")
lib = N.load(os.environ["TIDE_PROBE_LIB"]) if os.environ.get("TIDE_PROBE_LIB") else N.load()
ws = D.workspace().data_ptr()
s = torch.cuda.current_stream().cuda_stream


def launch():
    lib.tide_route(h.data_ptr(), d, n, None, n, d, N.BF16, None, wd.data_ptr(), wu.data_ptr(), b,
                   1e-6, 0.5, 3, scores.data_ptr(), None, mask.data_ptr(), ei.data_ptr(),
                   ci.data_ptr(), 0, None, counts.data_ptr(), ws, s)


for _ in range(20):
    launch()
torch.cuda.synchronize()
q = ("clocks.sm,power.draw,power.limit,clocks_event_reasons.sw_power_cap,"
     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,temperature.gpu")
p = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                      "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 0
t_end = time.time() + 3.0
while time.time() < t_end:
    for _ in range(200):
        launch()
    reps += 200
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
p.terminate()
out = p.communicate()[0].strip().splitlines()
print(f"{'zero' if zero else 'random'} data: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/launch over {reps}")
for ln in out[len(out) // 3: len(out) // 3 + 8]:
    print("  ", ln)
