#!/usr/bin/env python
"""Reduced-size launches of every product kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py

Each case runs the public API on small shapes (the sanitizers serialise and
instrument every access) and checks the result against the oracle, so a run
that passes both the tool and the checks covers the look-back, PDL, DSMEM
cluster and TMA/tcgen05 protocols of: the persistent tcgen05 router (K1),
the split-K cluster router (K1s), the peeling chain with its tail + resolve
kernels, the decode-step kernel, the CUDA-core f32 router, standalone
compaction with row gather, exit projection / select_project and the
labeller; round 2: K1's pair slots, the 3xTF32 f32 router, the wide chain
tail, the tensor-core LM head (via posthoc_select), the exit codec.
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_21365_b200 as P  # noqa: E402
from oracle import tide_oracle as O  # noqa: E402


def case_route(split, n, d, dt=torch.bfloat16):
    os.environ["TIDE_SPLIT"] = split
    g = np.random.Generator(np.random.PCG64(n + d))
    r = O.make_router(d, 128, 3, g)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32),
                   "f32" if dt == torch.float32 else "bf16")
    out = P.route(torch.from_numpy(h).cuda().to(dt), P.Router(3, r.w_down, r.w_up), theta=0.5,
                  want_logits=True, want_indices=True)
    torch.cuda.synchronize()
    _, t, m = O.route_logits(h, r)
    rt = 1e-5 if dt == torch.float32 else 2e-2
    assert O.logits_close(out["logits"].cpu().numpy(), t, m, rt).all()
    e, _ = O.compact_indices(out["mask"].cpu().numpy())
    assert np.array_equal(out["exiting_indices"].cpu().numpy(), e)
    os.environ.pop("TIDE_SPLIT", None)


def case_chain(n, d, L, theta):
    os.environ["TIDE_CHAIN_GRAPHS"] = "0"
    g = np.random.Generator(np.random.PCG64(L))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, 128, k, g, scale=0.15) for k in ckpts}
    host = [O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
            for _ in range(L + 1)]
    states = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in host]
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    got = P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=theta)).cpu().numpy()
    scores, exc = {}, np.zeros(n, bool)
    for k in ckpts:
        s, t, m = O.route_logits(host[k + 1], routers[k])
        scores[k] = s
        exc |= np.abs(t - O.logit_of(theta)) <= 2e-2 * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, theta)
    assert np.all((got == want) | exc)
    # decode step (every checkpoint in one launch) on the first rows; skipped
    # by SANITIZE_NO_DECODE=1 (under racecheck its cluster peers run so slowly
    # that the spin-limit trap fires; the decode has its own racecheck run)
    if os.environ.get("SANITIZE_NO_DECODE") != "1":
        dec = [s[:8].contiguous() for s in states]
        got8 = P.select_exits(dec, bank, P.RuntimeConfig(exit_threshold=theta)).cpu().numpy()
        assert np.all((got8 == want[:8]) | exc[:8])
    os.environ.pop("TIDE_CHAIN_GRAPHS", None)
    return states, bank, host


def case_project_label(states, bank, host):
    L = bank.num_layers
    d = host[0].shape[1]
    g = np.random.Generator(np.random.PCG64(5))
    head = P.OutputHead(L, d, g.standard_normal(d).astype(np.float32),
                        (g.standard_normal((64, d)) * 0.05).astype(np.float32))
    logits, exits = P.posthoc_select(head, states, bank, P.RuntimeConfig(exit_threshold=0.6))
    torch.cuda.synchronize()
    # compaction with the row gather, on a host mask
    mask = (np.arange(host[1].shape[0]) % 3 == 0)
    res = P.batch_compact(host[1], mask)
    e, c = O.compact_indices(mask.astype(np.uint8))
    assert np.array_equal(res.exiting_indices, e) and np.array_equal(res.continuing_indices, c)
    assert np.array_equal(res.exiting, host[1][e])
    # labeller over the checkpoints vs the final capture
    cs = P.CollectedStates({k: states[k + 1] for k in bank.checkpoints}, states[L],
                           host[0].shape[0], "x")
    ds = P.compute_labels(cs, 0.5)
    assert ds is not None


def case_round2():
    """Kernels added in round 2: K1 pair slots (dense whole-tile launch), the
    f32 3xTF32 route (forced at a small shape), the wide chain tail (theta >=
    0.9), the exit codec + global compaction (the multi-GPU exchange)."""
    case_route("0", 38400, 128)          # K1 pair slots: >= 148 x 256 rows, whole tiles
    os.environ["TIDE_F32_TC"] = "1"
    case_route("0", 600, 256, torch.float32)   # 3xTF32, segmented accumulators
    os.environ.pop("TIDE_F32_TC", None)
    os.environ["TIDE_SPECULATIVE"] = "0"
    case_chain(700, 256, 24, 0.95)       # link 1 + the wide tail + resolve
    os.environ.pop("TIDE_SPECULATIVE", None)
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N
    lib = N.load()
    s = Dv.stream_handle(torch.device("cuda", 0))
    lay = torch.randint(-1, 30, (5000,), dtype=torch.int64, device="cuda")
    code = torch.empty(5000, dtype=torch.uint8, device="cuda")
    N.check(lib.tide_exit_encode(lay.data_ptr(), 5000, code.data_ptr(), s), "encode")
    idx = torch.empty(5000, dtype=torch.int64, device="cuda")
    cnt = torch.empty(2, dtype=torch.int64, device="cuda")
    N.check(lib.tide_compact(code.data_ptr(), 5000, None, None, 0, None, 0, 0, 0, idx.data_ptr(),
                             None, None, None, cnt.data_ptr(), Dv.workspace().data_ptr(), s),
            "compact")
    torch.cuda.synchronize()
    want = np.flatnonzero(lay.cpu().numpy() >= 0)
    assert np.array_equal(idx[: int(cnt[0])].cpu().numpy(), want)


def case_k1m():
    """K1m (the whole per-token chain in one launch, exit map by atomic
    minimum), dense with pair slots and gathered; K1 with several row groups
    per CTA (the slot-release protocol), pair and single slots."""
    os.environ["TIDE_SPECULATIVE"] = "1"
    case_chain(1000, 512, 40, 0.6)      # dense K1m, ragged n, 10 checkpoints
    os.environ.pop("TIDE_SPECULATIVE", None)
    os.environ["TIDE_K1_GRID"] = "4"    # K1 as if on 4 SMs: several groups per CTA
    for pair in ("1", "0"):
        os.environ["TIDE_K1_PAIRSLOT"] = pair
        case_route("0", 4 * 1152, 128)  # 9 tiles per CTA: three groups each
    os.environ.pop("TIDE_K1_PAIRSLOT", None)
    os.environ.pop("TIDE_K1_GRID", None)


def case_round1():
    case_route("0", 2000, 1024)          # persistent tcgen05 K1 (ragged tail)
    case_route("16", 1000, 2048)         # split-K cluster kernel
    case_route("0", 700, 768, torch.float32)  # CUDA-core f32 router
    os.environ["TIDE_SPECULATIVE"] = "0"  # the peeling chain, not K1m
    st, bank, host = case_chain(1500, 512, 32, 0.55)  # peeling links + tail + resolve
    os.environ.pop("TIDE_SPECULATIVE", None)
    case_project_label(st, bank, host)


def case_late():
    """Kernels changed late in round 2: the staged exit projection /
    select_project (bf16 and f32 rows, ragged d), the CTA-pair LM head (via
    posthoc_select), batch_compact's parallel row gather."""
    os.environ["SANITIZE_NO_DECODE"] = "1"
    st, bank, host = case_chain(300, 772, 12, 0.6)
    os.environ.pop("SANITIZE_NO_DECODE", None)
    case_project_label(st, bank, host)
    g = np.random.Generator(np.random.PCG64(9))
    for dt in (torch.float32, torch.bfloat16):
        rows = torch.from_numpy(g.standard_normal((200, 1000), dtype=np.float32)).cuda().to(dt)
        gain = g.standard_normal(1000).astype(np.float32)
        pos = torch.arange(0, 400, 2, dtype=torch.int64, device="cuda")
        out = torch.zeros((400, 1000), device="cuda")
        P.exit_projection(rows, gain, 1e-6, pos, out)
        want = np.zeros((400, 1000), np.float32)
        O.exit_projection(rows.float().cpu().numpy(), gain, 1e-6, pos.cpu().numpy(), want)
        assert np.array_equal(out.cpu().numpy(), want)


CASES = {"round1": case_round1, "round2": case_round2, "k1m": case_k1m, "late": case_late}


def main():
    """python tools/sanitize_cases.py [round1|round2|k1m ...] (default: all)"""
    assert torch.cuda.is_available()
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
        print(f"sanitize cases ok: {name}")


if __name__ == "__main__":
    main()
