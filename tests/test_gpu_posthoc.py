"""GPU parity: posthoc_select (per-token peeling chain, batch-unanimous, decode
path) vs the reference golden exit maps / logits — restates
pkg/tests/test_runtime.py:42-147 against the device path, plus configs 2, 3
and 5 shapes against the oracle."""

import numpy as np
import pytest
import torch

import paper_2603_21365_b200 as P
from oracle import tide_oracle as O
from tests.golden.cases import (bank_from_golden, digest, posthoc_cases, posthoc_states,
                                rigged_router_arrays, stored_digest)
from tests.gpu_helpers import RTOL, excused_rows, need_gpu

pytestmark = pytest.mark.gpu


def _bank(g, bname):
    ckpts, eps, ws = bank_from_golden(g, bname)
    return P.make_bank(ws, num_layers=12, interval=4, eps=eps), ckpts, eps, ws


def _head(g):
    return P.OutputHead(12, 64, g["final_norm"], g["lm_head"])


def test_golden_exit_maps_and_logits(golden_posthoc):
    need_gpu()
    g = golden_posthoc
    head = _head(g)
    banks = {b: _bank(g, b) for b in ("rigged", "trained")}
    cache = {}
    n_checked = 0
    for idx, (seed, n, zero_row, bname, theta, mode, k_min) in enumerate(posthoc_cases(g)):
        key = (seed, n, zero_row)
        if key not in cache:
            cache[key] = posthoc_states(seed, n, zero_row)
        states = cache[key]
        assert digest(*states) == stored_digest(g, f"c{idx}__digest")
        bank, ckpts, eps, ws = banks[bname]
        cfg = P.RuntimeConfig(exit_threshold=theta, mode=mode, k_min=k_min)
        logits, exits = P.posthoc_select(head, states, bank, cfg)
        want = g[f"c{idx}__exits"]
        routers = {k: O.OracleRouter(k, *ws[k]) for k in ckpts}
        exc = excused_rows(states, routers, theta, "f32", k_min)
        if mode == P.BATCH_UNANIMOUS and exc.any():
            exc[:] = True  # one excused row can flip the unanimous decision for all
        assert np.all((exits == want) | exc), (idx, exits, want)
        if f"c{idx}__logits" in g.files and not exc.any():
            np.testing.assert_allclose(logits, g[f"c{idx}__logits"], atol=1e-5, rtol=0)
        n_checked += 1
    assert n_checked == 200


def test_reference_runtime_semantics(golden_posthoc):
    """pkg/tests/test_runtime.py:52-137 on the device path."""
    need_gpu()
    g = golden_posthoc
    head = _head(g)
    rigged, _, _, _ = _bank(g, "rigged")
    rng = np.random.Generator(np.random.PCG64(1234))
    states = [rng.standard_normal((6, 64), dtype=np.float32) for _ in range(13)]
    base = O.lm_head_from_hidden(g["final_norm"], g["lm_head"], states[-1])
    for mode in P.MODES:
        logits, exits = P.posthoc_select(head, states, rigged,
                                         P.RuntimeConfig(exit_threshold=1.0, mode=mode))
        assert np.all(exits == P.NO_EXIT)
        np.testing.assert_allclose(logits, base, atol=1e-5)
        logits, exits = P.posthoc_select(head, states, rigged,
                                         P.RuntimeConfig(exit_threshold=0.5, mode=mode))
        assert np.all(exits == 7)
        np.testing.assert_allclose(
            logits, O.lm_head_from_hidden(g["final_norm"], g["lm_head"], states[8]), atol=1e-5)
    _, exits = P.posthoc_select(head, states, rigged, P.RuntimeConfig(exit_threshold=0.5, k_min=8))
    assert np.all(exits == P.NO_EXIT)
    states[8][2] = 0.0
    _, per_token = P.posthoc_select(head, states, rigged, P.RuntimeConfig(exit_threshold=0.5))
    want = np.full(6, 7)
    want[2] = P.NO_EXIT
    np.testing.assert_array_equal(per_token, want)
    _, unanimous = P.posthoc_select(head, states, rigged,
                                    P.RuntimeConfig(exit_threshold=0.5, mode=P.BATCH_UNANIMOUS))
    assert np.all(unanimous == P.NO_EXIT)
    logits, exits = P.posthoc_select(head, states, None, P.RuntimeConfig())
    assert np.all(exits == P.NO_EXIT)
    with pytest.raises(ValueError, match="hidden states"):
        P.posthoc_select(head, states[:-1], rigged, P.RuntimeConfig())
    with pytest.raises(ValueError, match="width"):
        P.posthoc_select(head, [s[:, :32] for s in states], rigged, P.RuntimeConfig())


def test_reference_bank_object_is_accepted(golden_posthoc):
    """Duck-typed drop-in: an object with the reference RouterBank's fields."""
    need_gpu()
    g = golden_posthoc
    ours, ckpts, eps, ws = _bank(g, "trained")

    class RefLikeBank:  # fields of ee/calibration.py:351-382
        pass

    b = RefLikeBank()
    for f in ("hidden_dim", "bottleneck", "interval", "tau", "eps", "num_layers", "routers"):
        setattr(b, f, getattr(ours, f))
    b.checkpoints = ours.checkpoints
    states = posthoc_states(1236, 300)
    cfg = P.RuntimeConfig(exit_threshold=0.5)
    _, e1 = P.posthoc_select(_head(g), states, ours, cfg)
    _, e2 = P.posthoc_select(_head(g), states, b, cfg)
    np.testing.assert_array_equal(e1, e2)


def _big_case(L, d, n, dtype, seed, scale=0.1, b=128):
    """Synthetic capture + bank at a BASELINE config shape (device tensors)."""
    g = np.random.Generator(np.random.PCG64(seed))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, b, k, g, scale=scale) for k in ckpts}
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16}[dtype]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    states = [None] * (L + 1)
    for k in list(ckpts) + [L - 1]:
        states[k + 1] = torch.randn((n, d), generator=gen, device="cuda").to(tdt)
    for i in range(L + 1):
        if states[i] is None:
            states[i] = states[L]  # never read by the exit path
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    head = P.OutputHead(L, d, np.ones(d, np.float32),
                        (g.standard_normal((256, d)) * 0.02).astype(np.float32))
    return ckpts, routers, states, bank, head


@pytest.mark.parametrize("theta", [0.5, 0.85, 1.0])
@pytest.mark.parametrize("mode", [P.PER_TOKEN, P.BATCH_UNANIMOUS])
def test_config2_prefill_shape(theta, mode):
    """DeepSeek-8B shape: L=32 (8 checkpoints), d=4096, 4,096 tokens, bf16."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(32, 4096, 4096, "bf16", 2)
    cfg = P.RuntimeConfig(exit_threshold=theta, mode=mode)
    logits, exits = P.posthoc_select(head, states, bank, cfg)
    host = {k + 1: states[k + 1].float().cpu().numpy() for k in ckpts}
    scores, exc = {}, np.zeros(4096, bool)
    for k in ckpts:
        s, t, m = O.route_logits(host[k + 1], routers[k])
        scores[k] = s
        if theta < 1.0:
            exc |= np.abs(t - O.logit_of(theta)) <= RTOL["bf16"] * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, theta, 0, mode)
    got = exits.cpu().numpy()
    if mode == P.BATCH_UNANIMOUS and exc.any():
        exc[:] = True
    assert np.all((got == want) | exc)
    if theta == 1.0:
        assert np.all(got == P.NO_EXIT)
    # logits: final-norm of the chosen layer's row through the LM head
    fin = states[32].float().cpu().numpy()
    rows = np.stack([host[int(k) + 1][i] if k >= 0 else fin[i] for i, k in enumerate(got)])
    ref = O.lm_head_from_hidden(np.ones(4096, np.float32), head.lm_head, rows)
    np.testing.assert_allclose(logits.cpu().numpy(), ref, atol=2e-4, rtol=1e-4)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("mode", [P.PER_TOKEN, P.BATCH_UNANIMOUS])
@pytest.mark.parametrize("n", [1, 8, 16])
def test_config3_decode_step(dtype, mode, n):
    """Qwen3-8B shape decode: L=36 (9 checkpoints), d=4096, <=16 rows, one launch."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(36, 4096, n, dtype, 3, scale=0.3)
    for theta in (0.5, 0.85, 1.0):
        cfg = P.RuntimeConfig(exit_threshold=theta, mode=mode)
        exits = P.select_exits(states, bank, cfg).cpu().numpy()
        scores, exc = {}, np.zeros(n, bool)
        for k in ckpts:
            s, t, m = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
            scores[k] = s
            if theta < 1.0:
                exc |= np.abs(t - O.logit_of(theta)) <= RTOL[dtype] * np.maximum(np.abs(t), m)
        want = O.first_exit_from_scores(scores, theta, 0, mode)
        if mode == P.BATCH_UNANIMOUS and exc.any():
            exc[:] = True
        assert np.all((exits == want) | exc), (theta, exits, want)


def test_config5_shard_shape_peeling_chain():
    """70B shape, one 8,192-token shard: d=8192, 20 checkpoints, bf16."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(80, 8192, 8192, "bf16", 5, scale=0.06)
    exits = P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=0.7)).cpu().numpy()
    scores, exc = {}, np.zeros(2048, bool)
    for k in ckpts:
        s, t, m = O.route_logits(states[k + 1][:2048].float().cpu().numpy(), routers[k])
        scores[k] = s
        exc |= np.abs(t - O.logit_of(0.7)) <= RTOL["bf16"] * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, 0.7)
    assert np.all((exits[:2048] == want) | exc)
    assert (exits >= 0).mean() > 0.05  # the chain actually peels rows


def test_rigged_hot_bf16_device_exact():
    """Rigged routers saturate to exactly 1.0 / 0.0 on the tensor-core path too."""
    need_gpu()
    d = 64
    L = 12
    routers = {k: rigged_router_arrays(d, hot=(k == 7)) for k in (3, 7, 11)}
    bank = P.make_bank(routers, num_layers=L)
    g = np.random.Generator(np.random.PCG64(9))
    states = [torch.from_numpy(O.round_to(g.standard_normal((500, d), dtype=np.float32), "bf16"))
              .cuda().to(torch.bfloat16) for _ in range(L + 1)]
    states[8][17] = 0.0  # zero row scores exactly 0.5 at layer 7 -> never exits
    head = P.OutputHead(L, d, np.ones(d, np.float32), np.eye(d, dtype=np.float32))
    _, exits = P.posthoc_select(head, states, bank, P.RuntimeConfig(exit_threshold=0.5))
    e = exits.cpu().numpy()
    assert e[17] == P.NO_EXIT and np.all(np.delete(e, 17) == 7)
    _, exits = P.posthoc_select(head, states, bank, P.RuntimeConfig(exit_threshold=1.0))
    assert np.all(exits.cpu().numpy() == P.NO_EXIT)


@pytest.mark.parametrize("mode", [P.PER_TOKEN, P.BATCH_UNANIMOUS])
def test_decode_step_object_matches_select_exits(mode):
    """DecodeStep (bound once, static buffers) == select_exits on the same
    buffers, including after the buffers are rewritten in place."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(36, 4096, 8, "bf16", 31, scale=0.3)
    cfg = P.RuntimeConfig(exit_threshold=0.55, mode=mode)
    step = P.DecodeStep(states, bank, cfg)
    for it in range(3):
        if it:
            g = torch.Generator(device="cuda")
            g.manual_seed(100 + it)
            for k in ckpts:
                states[k + 1].copy_(torch.randn(states[k + 1].shape, generator=g,
                                                device="cuda").to(states[k + 1].dtype))
        got = step().clone()
        want = P.select_exits(states, bank, cfg)
        assert torch.equal(got, want)


@pytest.mark.parametrize("d,n,L,scale,theta", [(4096, 4096, 32, 0.1, 0.5), (8192, 2048, 40, 0.06, 0.7),
                                               (4096, 1000, 24, 0.2, 0.55), (4096, 1000, 24, 0.2, 1.0),
                                               (2048, 700, 28, 0.2, 0.6)])
def test_chain_tail_matches_oracle_and_links(d, n, L, scale, theta, monkeypatch):
    """The chain tail (one launch for the remaining checkpoints once few rows
    are live) gives the oracle's first-exit map (band rule), as the plain links do."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(L, d, n, "bf16", 7 + d + n, scale=scale)
    cfg = P.RuntimeConfig(exit_threshold=theta)
    scores, exc = {}, np.zeros(n, bool)
    for k in ckpts:
        s, t, m = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
        scores[k] = s
        exc |= np.abs(t - O.logit_of(theta)) <= RTOL["bf16"] * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, theta)
    out = {}
    # wide tail right after link 1 / links + small tail / plain links (peeling),
    # and the speculative one-launch K1m form
    monkeypatch.setenv("TIDE_SPECULATIVE", "0")
    for wide, tail in (("1", "1"), ("0", "1"), ("0", "0")):
        monkeypatch.setenv("TIDE_TAIL_WIDE", wide)
        monkeypatch.setenv("TIDE_CHAIN_TAIL", tail)
        got = P.select_exits(states, bank, cfg).cpu().numpy()
        assert np.all((got == want) | exc), (wide, tail)
        out[wide + tail] = got
    # a two-checkpoint speculative window, then the links (+ tail)
    monkeypatch.setenv("TIDE_TAIL_WIDE", "0")
    monkeypatch.setenv("TIDE_CHAIN_TAIL", "1")
    monkeypatch.setenv("TIDE_WINDOW", "2")
    out["win"] = P.select_exits(states, bank, cfg).cpu().numpy()
    monkeypatch.delenv("TIDE_WINDOW")
    assert np.all((out["win"] == want) | exc)
    monkeypatch.setenv("TIDE_SPECULATIVE", "1")
    out["spec"] = P.select_exits(states, bank, cfg).cpu().numpy()
    assert np.all((out["spec"] == want) | exc)
    assert np.all((out["11"] == out["00"]) | exc)
    assert np.all((out["01"] == out["00"]) | exc)
    assert np.all((out["spec"] == out["00"]) | exc)
    if theta == 1.0:
        assert all(np.all(v == P.NO_EXIT) for v in out.values())


@pytest.mark.parametrize("variant", [{"TIDE_DECODE_CLUSTER": "0"}, {"TIDE_DECODE_TMA": "0"},
                                     {"TIDE_DECODE_PACKED": "0"}, {"TIDE_PDL": "0"},
                                     {"TIDE_DECODE_CLUSTER": "0", "TIDE_DECODE_TMA": "0"}])
def test_decode_step_fallback_paths(variant, monkeypatch):
    """The global-ticket reduction and the cp.async W path give the same exit
    map as the default (cluster + TMA) decode kernel."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(36, 4096, 8, "bf16", 41, scale=0.3)
    cfg = P.RuntimeConfig(exit_threshold=0.5)
    want = P.select_exits(states, bank, cfg)
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    got = P.select_exits(states, bank, cfg)
    scores, exc = {}, np.zeros(8, bool)
    for k in ckpts:
        s_, t, m = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
        exc |= np.abs(t - O.logit_of(0.5)) <= RTOL["bf16"] * np.maximum(np.abs(t), m)
    assert np.all((got.cpu().numpy() == want.cpu().numpy()) | exc)


@pytest.mark.parametrize("d,n,L,scale,theta", [(4096, 4096, 32, 0.1, 0.5), (4096, 1000, 24, 0.2, 1.0),
                                               (8192, 2048, 40, 0.06, 0.7)])
@pytest.mark.parametrize("wide", ["1", "0", "spec"])
def test_chain_captured_in_cuda_graph(d, n, L, scale, theta, wide, monkeypatch):
    """select_exits captured in a CUDA graph (link 1 + the wide tail, or the
    links with the ones after the small chain tail in a conditional node the
    tail switches off, or the speculative K1m launch) == eager, on replays
    with new capture contents."""
    need_gpu()
    monkeypatch.setenv("TIDE_SPECULATIVE", "1" if wide == "spec" else "0")
    monkeypatch.setenv("TIDE_TAIL_WIDE", "1" if wide == "spec" else wide)
    ckpts, routers, states, bank, head = _big_case(L, d, n, "bf16", 90 + n, scale=scale)
    cfg = P.RuntimeConfig(exit_threshold=theta)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        P.select_exits(states, bank, cfg)  # warm caches (weights, plans) outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            out = P.select_exits(states, bank, cfg)
    torch.cuda.synchronize()
    for rep in range(3):
        if rep:
            gen = torch.Generator(device="cuda")
            gen.manual_seed(500 + rep)
            for k in ckpts:
                states[k + 1].copy_(torch.randn(states[k + 1].shape, generator=gen,
                                                device="cuda").to(states[k + 1].dtype))
            torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        want = P.select_exits(states, bank, cfg)
        assert torch.equal(out, want), rep


@pytest.mark.parametrize("d,n,L,scale,theta", [(4096, 4096, 32, 0.1, 0.5), (8192, 2048, 40, 0.06, 0.7)])
def test_eager_chain_graph_cache(d, n, L, scale, theta, monkeypatch):
    """Repeated eager select_exits calls with the same capture buffers replay a
    recorded chain: same exit map as the uncached path, new contents of the
    buffers are read, a returned map is not overwritten by the next call."""
    need_gpu()
    from paper_2603_21365_b200 import runtime as R
    ckpts, routers, states, bank, head = _big_case(L, d, n, "bf16", 300 + n, scale=scale)
    cfg = P.RuntimeConfig(exit_threshold=theta)
    R._chain_graphs.entries.clear()
    first = P.select_exits(states, bank, cfg)     # eager, counted
    second = P.select_exits(states, bank, cfg)    # recorded + replayed
    third = P.select_exits(states, bank, cfg)     # replayed
    assert len(R._chain_graphs.entries) == 1
    assert next(iter(R._chain_graphs.entries.values()))[1] is not None
    assert torch.equal(first, second) and torch.equal(first, third)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(77)
    for k in ckpts:
        states[k + 1].copy_(torch.randn(states[k + 1].shape, generator=gen,
                                        device="cuda").to(states[k + 1].dtype))
    replayed = P.select_exits(states, bank, cfg)
    monkeypatch.setenv("TIDE_CHAIN_GRAPHS", "0")
    eager = P.select_exits(states, bank, cfg)
    assert torch.equal(replayed, eager)
    assert torch.equal(third, first)  # earlier results are copies


@pytest.mark.parametrize("n,d,L,theta", [(2048, 768, 12, 0.5), (3000, 512, 24, 0.55),
                                         (500, 772, 16, 1.0)])
def test_f32_chain_all_checkpoints_at_once(n, d, L, theta, monkeypatch):
    """f32 rows, few of them: one CUDA-core launch scores every checkpoint and
    the resolve kernel picks the first firing one — the same exit map as the
    peeling links (and the oracle, to the f32 band)."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(n + d + L))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in ckpts}
    states = [torch.from_numpy(g.standard_normal((n, d), dtype=np.float32)).cuda()
              for _ in range(L + 1)]
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    cfg = P.RuntimeConfig(exit_threshold=theta)
    scores, exc = {}, np.zeros(n, bool)
    for k in ckpts:
        s_, t, m = O.route_logits(states[k + 1].cpu().numpy(), routers[k])
        scores[k] = s_
        exc |= np.abs(t - O.logit_of(theta)) <= RTOL["f32"] * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, theta)
    monkeypatch.setenv("TIDE_CHAIN_GRAPHS", "0")
    got = P.select_exits(states, bank, cfg).cpu().numpy()
    monkeypatch.setenv("TIDE_CHAIN_TAIL", "0")
    links = P.select_exits(states, bank, cfg).cpu().numpy()
    assert np.all((got == want) | exc) and np.all((links == want) | exc)
    assert np.array_equal(got, links)
    if theta == 1.0:
        assert np.all(got == P.NO_EXIT)


def test_chain_cache_host_inputs_and_router_swap(monkeypatch):
    """The replay cache with numpy (host) captures — fresh device copies every
    call, possibly at recycled addresses — and with a router replaced in the
    bank between calls: always the uncached result."""
    need_gpu()
    from paper_2603_21365_b200 import runtime as R
    ckpts, routers, states, bank, head = _big_case(24, 1024, 600, "bf16", 611, scale=0.2)
    host = [s.float().cpu().numpy() for s in states]
    cfg = P.RuntimeConfig(exit_threshold=0.55)
    R._chain_graphs.entries.clear()

    def uncached(st, bk):
        monkeypatch.setenv("TIDE_CHAIN_GRAPHS", "0")
        try:
            return P.select_exits(st, bk, cfg)
        finally:
            monkeypatch.delenv("TIDE_CHAIN_GRAPHS")

    g = np.random.Generator(np.random.PCG64(5))
    for it in range(4):
        if it == 2:  # new data in the host arrays
            for k in ckpts:
                host[k + 1] = g.standard_normal(host[k + 1].shape).astype(np.float32)
        assert torch.equal(P.select_exits(host, bank, cfg), uncached(host, bank)), it
    # replace one router (new object, new weights): a new key, a new recording
    k0 = ckpts[1]
    r = O.make_router(1024, 128, k0, g, scale=0.2)
    bank.routers[k0] = P.Router(layer=k0, w_down=r.w_down, w_up=r.w_up)
    for it in range(3):
        assert torch.equal(P.select_exits(states, bank, cfg), uncached(states, bank)), it


@pytest.mark.parametrize("mode", [P.PER_TOKEN, P.BATCH_UNANIMOUS])
@pytest.mark.parametrize("d,n", [(1024, 16), (512, 13), (2048, 3), (8192, 16)])
def test_decode_step_cluster_row_owners(mode, d, n):
    """Decode shapes whose cluster split leaves several rows per rank (small
    d -> few slice-CTAs) or idle ranks (n < S), against the oracle; scores /
    logits outputs and the exit count of the C ABI on the same launch."""
    need_gpu()
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N
    from paper_2603_21365_b200 import runtime as R
    ckpts, routers, states, bank, head = _big_case(36, d, n, "bf16", 77 + d + n, scale=0.3)
    for theta in (0.5, 0.85):
        cfg = P.RuntimeConfig(exit_threshold=theta, mode=mode)
        exits = P.select_exits(states, bank, cfg).cpu().numpy()
        scores, exc = {}, np.zeros(n, bool)
        for k in ckpts:
            s_, t, m = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
            scores[k] = s_
            exc |= np.abs(t - O.logit_of(theta)) <= RTOL["bf16"] * np.maximum(np.abs(t), m)
        want = O.first_exit_from_scores(scores, theta, 0, mode)
        if mode == P.BATCH_UNANIMOUS and exc.any():
            exc[:] = True
        assert np.all((exits == want) | exc), (theta, exits, want)
    # the raw C entry with every output: scores / logits / exit count
    code = N.BF16
    plan = R._decode_plan(bank, list(ckpts), code, states[0].device)
    C = len(ckpts)
    sc = torch.empty(C * n, dtype=torch.float32, device="cuda")
    lg = torch.empty(C * n, dtype=torch.float32, device="cuda")
    ex = torch.empty(n, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    lib = N.load()
    s = Dv.stream_handle()
    N.check(lib.tide_route_decode_ex(
        N.ptr_array([states[k + 1].data_ptr() for k in ckpts]), C, d, n, d, code, plan[0],
        plan[1], 128, plan[2], 1e-6, 0.5, 0, N.MODE_PER_TOKEN if mode == P.PER_TOKEN else
        N.MODE_BATCH_UNANIMOUS, sc.data_ptr(), lg.data_ptr(), ex.data_ptr(), cnt.data_ptr(),
        Dv.workspace().data_ptr(), plan[3], s), "decode")
    torch.cuda.synchronize()
    sc, lg, ex = sc.cpu().numpy().reshape(C, n), lg.cpu().numpy().reshape(C, n), ex.cpu().numpy()
    for i, k in enumerate(ckpts):
        s_ref, t_ref, m_ref = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
        assert O.logits_close(lg[i], t_ref, m_ref, RTOL["bf16"]).all()
        np.testing.assert_array_equal(sc[i], np.array([O._sigma64(float(v)) for v in lg[i]],
                                                      np.float32))
    assert int(cnt[0]) == int((ex >= 0).sum())


def _multi_call(states, bank, ckpts, n, d, code, row_idx=None, n_live=None, rows_total=None):
    """tide_route_multi through the C ABI: exit map over every checkpoint."""
    from paper_2603_21365_b200 import _device as D, _native as N
    from paper_2603_21365_b200.router_ops import device_weights
    lib = N.load()
    dev = torch.device("cuda", 0)
    wts = [device_weights(bank.routers[k], code, dev) for k in ckpts]
    out = torch.full((n,), P.NO_EXIT, dtype=torch.int64, device=dev)
    scratch = torch.empty(len(ckpts) * n, dtype=torch.float32, device=dev)
    n_dev = torch.tensor([n_live], dtype=torch.int64, device=dev) if row_idx is not None else None
    N.check(lib.tide_route_multi(
        N.ptr_array([states[k + 1].data_ptr() for k in ckpts]), len(ckpts), d, n,
        n_dev.data_ptr() if n_dev is not None else None, rows_total or n, d, code,
        row_idx.data_ptr() if row_idx is not None else None,
        N.ptr_array([w.data_ptr() for w, _ in wts]), N.ptr_array([u.data_ptr() for _, u in wts]),
        128, N.i64_array(ckpts), float(np.float32(bank.eps)), float(np.float32(0.6)),
        scratch.data_ptr(), out.data_ptr(), D.workspace(dev).data_ptr(), D.stream_handle(dev)),
        "tide_route_multi")
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("d,n,L,dtype", [(4096, 4096, 32, "bf16"), (4096, 1000, 24, "f16"),
                                         (8192, 700, 80, "bf16"), (768, 2048, 12, "bf16"),
                                         (2048, 300, 96, "bf16")])
def test_route_multi_dense_and_gathered(d, n, L, dtype):
    """K1m (tide_route_multi): dense over all rows and gathered over a live
    list (every other row, ragged count) == the oracle's per-token first-exit
    map over the same checkpoints (band rule); up to 24 checkpoints."""
    need_gpu()
    ckpts, routers, states, bank, head = _big_case(L, d, n, dtype, 11 + d + n, scale=0.15)
    ckpts = ckpts[:24]
    from paper_2603_21365_b200 import _native as N
    code = N.BF16 if dtype == "bf16" else N.F16
    host = {k: states[k + 1].float().cpu().numpy() for k in ckpts}
    scores, exc = {}, np.zeros(n, bool)
    for k in ckpts:
        s_, t, m = O.route_logits(host[k], routers[k])
        scores[k] = s_
        exc |= np.abs(t - O.logit_of(0.6)) <= RTOL[dtype] * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, 0.6)
    got = _multi_call(states, bank, ckpts, n, d, code)
    assert np.all((got == want) | exc)
    assert len(np.unique(got)) > 2  # rows leave at several checkpoints
    # gathered: the live list = odd rows (capacity n, live count n // 2)
    live = torch.arange(1, n, 2, dtype=torch.int64, device="cuda")
    idx = torch.zeros(n, dtype=torch.int64, device="cuda")
    idx[: live.numel()] = live
    gl = _multi_call(states, bank, ckpts, n, d, code, row_idx=idx, n_live=live.numel(), rows_total=n)
    sel = live.cpu().numpy()
    assert np.all((gl[sel] == want[sel]) | exc[sel])
    others = np.setdiff1d(np.arange(n), sel)
    assert np.all(gl[others] == P.NO_EXIT)


def test_speculative_chain_repeats_bitwise():
    """K1m (exit map by atomic minimum across CTAs): repeated select_exits
    calls on the same captures give the same exit map, with L2-thrashing
    writes in between (the minimum does not depend on arrival order)."""
    need_gpu()
    import os
    ckpts, routers, states, bank, head = _big_case(32, 4096, 4096, "bf16", 77, scale=0.1)
    cfg = P.RuntimeConfig(exit_threshold=0.6)
    os.environ["TIDE_SPECULATIVE"] = "1"
    try:
        want = P.select_exits(states, bank, cfg).clone()
        junk = torch.empty(1 << 26, device="cuda")
        for i in range(20):
            junk.fill_(float(i))
            assert torch.equal(P.select_exits(states, bank, cfg), want), i
    finally:
        os.environ.pop("TIDE_SPECULATIVE", None)
    assert (want >= 0).any() and len(torch.unique(want)) > 2


@pytest.mark.parametrize("d,n,L,b", [(776, 1000, 24, 128), (1024, 3000, 20, 256), (512, 700, 16, 64),
                                     (772, 500, 12, 128)])
def test_speculative_chain_odd_shapes(d, n, L, b, monkeypatch):
    """K1m through select_exits at shapes off the main configs: d not a
    multiple of 64 (partial last chunk), bottleneck 256 (two tiles per
    group) and 64 (narrow N), and d = 772 (not a multiple of 8: the policy
    must fall back to the peeling chain) -- the oracle's per-token map."""
    need_gpu()
    monkeypatch.setenv("TIDE_SPECULATIVE", "1")
    ckpts, routers, states, bank, head = _big_case(L, d, n, "bf16", 5 + d + b, scale=0.15, b=b)
    cfg = P.RuntimeConfig(exit_threshold=0.6)
    got = P.select_exits(states, bank, cfg).cpu().numpy()
    scores, exc = {}, np.zeros(n, bool)
    for k in ckpts:
        s_, t, m = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
        scores[k] = s_
        exc |= np.abs(t - O.logit_of(0.6)) <= RTOL["bf16"] * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, 0.6)
    assert np.all((got == want) | exc)
    monkeypatch.setenv("TIDE_SPECULATIVE", "0")
    peel = P.select_exits(states, bank, cfg).cpu().numpy()
    assert np.all((peel == want) | exc)


_FUZZ = [  # (n, d, L, dtype, theta, mode)
    (1, 64, 8, "bf16", 0.5, P.PER_TOKEN), (5, 772, 12, "f16", 0.6, P.PER_TOKEN),
    (16, 1000, 12, "bf16", 0.5, P.BATCH_UNANIMOUS), (17, 1000, 12, "bf16", 0.55, P.PER_TOKEN),
    (129, 256, 16, "f16", 0.5, P.PER_TOKEN), (300, 772, 20, "bf16", 0.95, P.PER_TOKEN),
    (1000, 96, 40, "bf16", 0.5, P.PER_TOKEN), (257, 4104, 8, "bf16", 0.6, P.PER_TOKEN),
    (2049, 512, 12, "f32", 0.5, P.PER_TOKEN), (640, 4096, 100, "bf16", 0.7, P.PER_TOKEN),
    (333, 2048, 12, "bf16", 1.0, P.PER_TOKEN), (4100, 128, 12, "f16", 0.5, P.BATCH_UNANIMOUS),
]


@pytest.mark.parametrize("n,d,L,dtype,theta,mode", _FUZZ)
def test_select_exits_policy_fuzz(n, d, L, dtype, theta, mode):
    """select_exits over shapes that steer every strategy (decode step, K1m,
    peeling links + tails, f32 tails, many checkpoints, d not a multiple of
    8, ragged n) against the oracle's first-exit map (band rule)."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(n * 7 + d + L))
    ckpts = O.checkpoint_layers(L, 4)
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in ckpts}
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    states = [torch.from_numpy(g.standard_normal((n, d), dtype=np.float32)).cuda().to(tdt)
              for _ in range(L + 1)]
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    cfg = P.RuntimeConfig(exit_threshold=theta, mode=mode)
    got = P.select_exits(states, bank, cfg).cpu().numpy()
    rt = 1e-5 if dtype == "f32" else RTOL["bf16"]
    scores, exc = {}, np.zeros(n, bool)
    for k in ckpts:
        s_, t, m = O.route_logits(states[k + 1].float().cpu().numpy(), routers[k])
        scores[k] = s_
        if theta < 1.0:
            exc |= np.abs(t - O.logit_of(theta)) <= rt * np.maximum(np.abs(t), m)
    want = O.first_exit_from_scores(scores, theta, 0, mode)
    if mode == P.BATCH_UNANIMOUS and exc.any():
        exc[:] = True
    assert np.all((got == want) | exc), (n, d, L, dtype, theta)
