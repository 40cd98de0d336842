"""Secondary timings for BASELINE.json configs 1-5 (bench.py --extra).

Each entry: device time (CUDA events on the launching stream, after warm-up)
of the B200 path for that config, with the algorithmic bytes it must move and
the resulting GB/s.  Synthetic inputs (torch cuda generator), random routers
N(0,1)*scale.  Not part of the driver's headline line.
"""

from __future__ import annotations

import numpy as np
import torch

import paper_2603_21365_b200 as P
from oracle import tide_oracle as O


def _time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def _case(L, d, n, dtype, seed, scale, b=128):
    g = np.random.Generator(np.random.PCG64(seed))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, b, k, g, scale=scale) for k in ckpts}
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    states = [None] * (L + 1)
    for k in list(ckpts) + [L - 1]:
        states[k + 1] = torch.randn((n, d), generator=gen, device="cuda").to(dtype)
    for i in range(L + 1):
        if states[i] is None:
            states[i] = states[L]
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    return ckpts, states, bank


def config2(theta=0.5):
    ckpts, states, bank = _case(32, 4096, 4096, torch.bfloat16, 2, 0.1)
    cfg = P.RuntimeConfig(exit_threshold=theta)
    exits = P.select_exits(states, bank, cfg)
    ms = _time(lambda: P.select_exits(states, bank, cfg))
    gms = _graph_time(lambda: P.select_exits(states, bank, cfg))
    # peeled bytes: every remaining row at every checkpoint
    e = exits.cpu().numpy()
    remaining, peeled = 4096, 0
    for k in ckpts:
        peeled += remaining * (4096 * 2 + 21)
        remaining -= int((e == k).sum())
    peeled += len(ckpts) * (128 * 4096 * 2 + 512)
    return {"config": "2: DeepSeek-8B prefill, L=32 (8 ckpts), d=4096, 4,096 tok, bf16, "
                      f"per-token theta={theta}",
            "ms_api": ms, "ms_graph": gms, "tokens_per_s": 4096 / (gms / 1e3),
            "peeled_bytes": peeled, "gbs_graph": peeled / (gms / 1e3) / 1e9,
            "exit_rate": float((e >= 0).mean()), **_strategy(ckpts, 4096, 4096, states, theta, gms)}


def _strategy(ckpts, n, d, states, theta, gms):
    """Which chain form select_exits took and the bytes it actually reads:
    speculative (K1m: every row at every checkpoint, 2 launches) or peeling
    (one link per checkpoint, live rows only)."""
    from paper_2603_21365_b200 import runtime as R
    spec = len(ckpts) <= R.MAX_MULTI_CKPTS and R._speculative(n, d, states[-1], theta, len(ckpts))
    if not spec:
        return {"strategy": "peeling", "launches": len(ckpts)}
    read = len(ckpts) * (n * (d * 2 + 4) + 128 * d * 2 + 512)
    return {"strategy": "speculative (K1m)", "launches": 2, "read_bytes": read,
            "gbs_read": read / (gms / 1e3) / 1e9}


def _graph_time(fn, reps=50, inner=1):
    """Device time of fn() replayed from a CUDA graph (no host work in the loop).
    `inner` calls are captured per graph so a short call (the one-launch decode
    step) is not timed against the graph-launch rate of the host."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(inner):
                fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / inner


def config3(mode=P.PER_TOKEN, dtype=torch.bfloat16):
    ckpts, states, bank = _case(36, 4096, 8, dtype, 3, 0.3)
    cfg = P.RuntimeConfig(exit_threshold=0.5, mode=mode)
    ms = _time(lambda: P.select_exits(states, bank, cfg), reps=50)
    gms = _graph_time(lambda: P.select_exits(states, bank, cfg), reps=20, inner=20)
    byts = len(ckpts) * (8 * 4096 * 2 + 128 * 4096 * 2)
    return {"config": f"3: Qwen3-8B decode, L=36 (9 ckpts), d=4096, 8 rows, {dtype}, {mode}",
            "us_per_step_api": ms * 1e3, "us_per_step_graph": gms * 1e3, "bytes": byts,
            "gbs_graph": byts / (gms / 1e3) / 1e9, "launches": 1}


def config4(n=1_024_000, d=4096, C=8):
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    fin = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    cks = {}
    for i in range(C + 1):
        t = fin if i == C else torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
        for r0 in range(0, n, 131072):
            r1 = min(n, r0 + 131072)
            t[r0:r1] = torch.randn((r1 - r0, d), generator=gen, device="cuda").to(torch.bfloat16)
        if i < C:
            cks[3 + 4 * i] = t
    ms = _time(lambda: P.label_tensors(cks, fin, 0.98, labels_dtype="u8"), reps=3, warm=1)
    byts = n * (C + 1) * d * 2 + n * C * 5
    out = {"config": f"4: calibration labeller, {n:,} tok x d={d} bf16, {C} ckpts + final",
           "ms": ms, "bytes": byts, "gbs": byts / (ms / 1e3) / 1e9}
    del fin, cks
    torch.cuda.empty_cache()
    return out


def config5(theta=0.7):
    ckpts, states, bank = _case(80, 8192, 8192, torch.bfloat16, 5, 0.06)
    cfg = P.RuntimeConfig(exit_threshold=theta)
    exits = P.select_exits(states, bank, cfg)
    ms = _time(lambda: P.select_exits(states, bank, cfg))
    gms = _graph_time(lambda: P.select_exits(states, bank, cfg))
    e = exits.cpu().numpy()
    remaining, peeled = 8192, 0
    for k in ckpts:
        peeled += remaining * (8192 * 2 + 21)
        remaining -= int((e == k).sum())
    return {"config": f"5: 70B prefill shard, L=80 (20 ckpts), d=8192, 8,192 tok/GPU, bf16, "
                      f"per-token theta={theta}",
            "ms_api": ms, "ms_graph": gms, "tokens_per_s": 8192 / (gms / 1e3),
            "peeled_bytes": peeled, "gbs_graph": peeled / (gms / 1e3) / 1e9,
            "exit_rate": float((e >= 0).mean()), **_strategy(ckpts, 8192, 8192, states, theta, gms)}


def config1():
    g = np.random.Generator(np.random.PCG64(42))
    ckpts = O.checkpoint_layers(12, 4)
    routers = {k: O.make_router(768, 128, k, g) for k in ckpts}
    states = [torch.from_numpy(g.standard_normal((2048, 768), dtype=np.float32)).cuda()
              for _ in range(13)]
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=12)
    cfg = P.RuntimeConfig(exit_threshold=0.5)
    ms = _time(lambda: P.select_exits(states, bank, cfg))
    gms = _graph_time(lambda: P.select_exits(states, bank, cfg))
    return {"config": "1: GPT-2-small shape, L=12 (3 ckpts), d=768, 2,048 tok, fp32 (CUDA-core "
                      "path, f32 products)", "ms_api": ms, "ms_graph": gms,
            "tokens_per_s": 2048 / (gms / 1e3)}


def training(n=65_536, d=4096, epochs=2):
    """GPU router training (§8f-4) on one checkpoint's calibration rows."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(6)
    x = torch.randn((n, d), generator=gen, device="cuda")
    y = (x[:, 0] > 0).to(torch.float32)
    cfg = P.CalibrationConfig(epochs=epochs, batch_size=1024, learning_rate=1e-3)
    P.train_router(x[:4096], y[:4096], 3, P.CalibrationConfig(epochs=1))  # warm-up
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    _, st = P.train_router(x, y, 3, cfg)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    return {"config": f"router training (GPU), {n:,} rows x d={d}, b=128, batch 1024, "
                      f"{epochs} epochs", "s_total": sec, "ms_per_epoch": sec / epochs * 1e3,
            "rows_per_s": n * epochs / sec, "accuracy": st.accuracy}


def lm_head(n=4096, d=4096, V=50257):
    """§8f-1: posthoc_select's LM head on tcgen05 (3 bf16 MMA terms, f32-grade)
    at GPT-2's vocabulary, against the f32 library GEMM it replaced."""
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N
    from paper_2603_21365_b200.runtime import split_bf16
    gen = torch.Generator(device="cuda")
    gen.manual_seed(8)
    a = torch.randn((n, d), generator=gen, device="cuda")
    w = torch.randn((V, d), generator=gen, device="cuda") * 0.02
    ah, al = split_bf16(a, d)
    bh, bl = split_bf16(w, d)
    ldo = (V + 3) // 4 * 4
    out = torch.empty((n, ldo), dtype=torch.float32, device="cuda")
    lib = N.load()
    s = Dv.stream_handle(torch.device("cuda", 0))

    def run(terms):
        return lambda: lib.tide_lm_head(ah.data_ptr(), al.data_ptr() if terms == 3 else None, d, n,
                                        d, bh.data_ptr(), bl.data_ptr() if terms == 3 else None,
                                        d, V, out.data_ptr(), ldo, s)
    ms3 = _time(run(3), reps=10)
    ms1 = _time(run(1), reps=10)
    torch.backends.cuda.matmul.allow_tf32 = False
    ms_lib = _time(lambda: a @ w.t(), reps=3, warm=1)
    flop = 2.0 * n * V * d
    return {"config": f"LM head (f8-1): logits [{n} x {V}] = rows [{n} x {d}] . W^T, f32-grade",
            "ms_3term": ms3, "tflops_3term_bf16_mma": 3 * flop / (ms3 / 1e3) / 1e12,
            "tflops_3term_f32_equiv": flop / (ms3 / 1e3) / 1e12,
            "ms_1term_bf16": ms1, "tflops_1term": flop / (ms1 / 1e3) / 1e12,
            "ms_torch_f32_sgemm": ms_lib, "speedup_3term_vs_sgemm": ms_lib / ms3}


def chain_sweep():
    """Peeling-chain configs 2 and 5 across thresholds, down to the worst case
    theta = 1.0 where no row ever exits and every link routes every row."""
    return ([config2(t) for t in (0.5, 0.7, 0.85, 1.0)]
            + [config5(t) for t in (0.5, 0.7, 0.85, 1.0)])


def dropin_numpy(n=65_536, d=4096, b=128):
    """The reference-facing call a user of earlyexit makes, unchanged:
    fused_layernorm_route(h, router) with h a host numpy f32 array and the
    scores returned as a host array (ee/router_ops.py:68-87) — pageable H2D
    of the f32 rows, the 3xTF32 tcgen05 kernel, D2H of the scores, all inside
    the wall-clock region.  Scores checked against the oracle on the first
    2,048 rows (1e-5 logit contract through the score: |ds| <= 1e-5 * 0.25 m
    is below f32 resolution here, so the check is the band rule on decisions)."""
    import time
    g = np.random.Generator(np.random.PCG64(5))
    h = g.standard_normal((n, d), dtype=np.float32)
    orouter = O.make_router(d, b, 3, g)
    router = P.Router(layer=3, w_down=orouter.w_down, w_up=orouter.w_up)
    for _ in range(2):
        P.fused_layernorm_route(h, router)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        s = P.fused_layernorm_route(h, router)
    wall = (time.perf_counter() - t0) / reps
    _, t_ref, m_ref = O.route_logits(h[:2048], orouter)
    ok = O.decision_band_ok(s[:2048] > np.float32(0.5), t_ref, m_ref, 0.5, 1e-5)
    return {"config": f"drop-in numpy API: fused_layernorm_route(h host f32 [{n} x {d}]) -> host scores",
            "ms_wall": wall * 1e3, "tokens_per_s": n / wall, "h2d_bytes": n * d * 4,
            "d2h_bytes": n * 4, "h2d_gbs": n * d * 4 / wall / 1e9,
            "decisions_ok_first_2048": bool(ok.all())}


def dropin_posthoc(L=32, d=4096, n=4096, V=50257, theta=0.5):
    """The reference-facing posthoc_select(model, hidden_states, bank, config)
    with host numpy f32 captures (L + 1 arrays [n, d]; config-2 shape) and a
    GPT-2-sized vocabulary, host logits [n, V] back — wall clock per call,
    uploads of the checkpoint + final captures, the exit chain, the staging,
    the tensor-core LM head and the 823 MB logits download inside."""
    import time
    g = np.random.Generator(np.random.PCG64(9))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, 128, k, g, scale=0.1) for k in ckpts}
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    base = g.standard_normal((n, d), dtype=np.float32)
    states = [base if i not in [k + 1 for k in ckpts] else
              g.standard_normal((n, d), dtype=np.float32) for i in range(L + 1)]
    head = P.OutputHead(L, d, np.ones(d, np.float32),
                        (g.standard_normal((V, d)) * 0.02).astype(np.float32))
    cfg = P.RuntimeConfig(exit_threshold=theta)
    P.posthoc_select(head, states, bank, cfg)  # device caches (LM head split) built once
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        logits, exits = P.posthoc_select(head, states, bank, cfg)
    wall = (time.perf_counter() - t0) / reps
    return {"config": f"drop-in posthoc_select: {L + 1} host f32 captures [{n} x {d}], "
                      f"{len(ckpts)} ckpts, vocab {V}, host logits back",
            "ms_wall": wall * 1e3, "tokens_per_s": n / wall,
            "h2d_bytes": (len(ckpts) + 1) * n * d * 4, "d2h_bytes": n * V * 4 + n * 8,
            "exit_rate": float((np.asarray(exits) >= 0).mean())}


def run_configs(hbm_gbs: float, bf16_tflops: float):
    """The BASELINE configs timed inside the driver's default bench run (N=1),
    each with its roofline fraction: HBM for the streaming paths (algorithmic
    / peeled bytes), bf16 tensor peak for the LM head."""
    out = []
    for fn in (config1, lambda: config2(0.5), lambda: config2(1.0), config3, config4,
               lambda: config5(0.5), lambda: config5(0.7), lambda: config5(1.0), lm_head,
               dropin_numpy, dropin_posthoc):
        try:
            r = fn()
        except Exception as e:  # report, do not hide
            out.append({"error": repr(e)[:300]})
            continue
        for k in ("gbs_graph", "gbs"):
            if k in r:
                r["hbm_frac"] = r[k] / hbm_gbs
        if "gbs_read" in r:
            r["hbm_frac_read"] = r["gbs_read"] / hbm_gbs
        if "tflops_3term_bf16_mma" in r:
            r["tensor_frac_3term"] = r["tflops_3term_bf16_mma"] / bf16_tflops
        out.append(r)
    return out


def run_extra(dev=None):
    out = []
    for fn in (config1, config2, config3,
               lambda: config3(P.BATCH_UNANIMOUS), lambda: config3(dtype=torch.float16),
               config5, config4, lm_head, training):
        try:
            out.append(fn())
        except Exception as e:  # report, do not hide
            out.append({"error": repr(e)})
    return out


if __name__ == "__main__":
    import json
    import sys
    if len(sys.argv) > 1 and sys.argv[1] == "lm":
        print(json.dumps(lm_head()), flush=True)
    elif len(sys.argv) > 1 and sys.argv[1] == "sweep":
        for r in chain_sweep():
            print(json.dumps(r), flush=True)
    else:
        for r in run_extra():
            print(json.dumps(r), flush=True)
