"""Device time of one K1 launch at the headline shape (65,536 x 4096 bf16),
back-to-back launches bracketed by CUDA events.  Run once per experiment
setting (TIDE_DEBUG_FLAGS / TIDE_K1_PAIR / TIDE_NW are read once per process):

    for f in 0 1 2 3 4; do TIDE_DEBUG_FLAGS=$f python tools/k1_probe.py; done
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_21365_b200 import _device as D, _native as N  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    d, b = 4096, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    h = torch.randn((n, d), generator=g, device="cuda").to(torch.bfloat16)
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
        N.check(lib.tide_route(h.data_ptr(), d, n, None, n, d, N.BF16, None, wd.data_ptr(),
                               wu.data_ptr(), b, 1e-6, 0.5, 3, scores.data_ptr(), None,
                               mask.data_ptr(), ei.data_ptr(), ci.data_ptr(), 0, None,
                               counts.data_ptr(), ws, s), "route")

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    alg = n * (d * 2 + 13) + b * d * 2 + b * 4
    env = {k: v for k, v in os.environ.items() if k.startswith("TIDE_")}
    print(json.dumps({"env": env, "n": n, "us": round(best, 2), "gbs": round(alg / best / 1e3, 1)}))


if __name__ == "__main__":
    main()
