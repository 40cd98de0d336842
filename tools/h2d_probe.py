"""Pinned host -> device copy rate of 512 MiB: one copy vs the same bytes split
over 2 / 4 streams (copy engines), CUDA events around the whole transfer."""
import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(main)
        part = n // k
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{k} stream(s): {best:.3f} ms  {n / best / 1e6:.1f} GB/s", flush=True)
