"""Regression tests for the round-1 advisor findings (shapes the one-launch
paths do not take, per-forward hook state, per-graph workspaces, capture
shape checks, device caches)."""

import gc

import numpy as np
import pytest
import torch
import torch.nn as nn

import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _device as D
from oracle import tide_oracle as O
from tests.gpu_helpers import RTOL, need_gpu


def _states_bank(n, d, L, ckpts, seed, dtype=torch.float32, scale=0.2, interval=1):
    g = np.random.Generator(np.random.PCG64(seed))
    routers = {k: O.make_router(d, 128, k, g, scale=scale) for k in ckpts}
    host = [O.round_to(g.standard_normal((n, d), dtype=np.float32),
                       "f32" if dtype == torch.float32 else "bf16") for _ in range(L + 1)]
    states = [torch.from_numpy(h).cuda().to(dtype) for h in host]
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L,
                       interval=interval)
    return routers, host, states, bank


def _want(routers, host, theta, dtype, n):
    scores, exc = {}, np.zeros(n, bool)
    for k, r in routers.items():
        s, t, m = O.route_logits(host[k + 1], r)
        scores[k] = s
        if theta < 1.0:
            exc |= np.abs(t - O.logit_of(theta)) <= RTOL[dtype] * np.maximum(np.abs(t), m)
    return O.first_exit_from_scores(scores, theta), exc


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,C", [(300, 66, 4), (300, 128, 40), (9, 64, 70), (200, 70, 70)])
def test_f32_shapes_outside_the_one_launch_kernels(n, d, C, monkeypatch):
    """d % 4 != 0 or more than 32 checkpoints (f32 tail) / more than 64
    (decode kernel): the chain takes them, same exit map as the oracle."""
    need_gpu()
    monkeypatch.setenv("TIDE_CHAIN_GRAPHS", "0")
    L = C
    ckpts = list(range(C))
    routers, host, states, bank = _states_bank(n, d, L, ckpts, n + d + C)
    assert tuple(bank.checkpoints) == tuple(ckpts)
    theta = 0.6
    want, exc = _want(routers, host, theta, "f32", n)
    got = P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=theta)).cpu().numpy()
    assert np.all((got == want) | exc)
    assert (got >= 0).any()


@pytest.mark.gpu
def test_bf16_chain_more_than_32_remaining_checkpoints(monkeypatch):
    """The chain tail takes at most 32 checkpoints; longer chains keep peeling."""
    need_gpu()
    monkeypatch.setenv("TIDE_CHAIN_GRAPHS", "0")
    n, d, C = 700, 256, 40
    routers, host, states, bank = _states_bank(n, d, C, list(range(C)), 9, torch.bfloat16,
                                               scale=0.1)
    want, exc = _want(routers, host, 0.9, "bf16", n)
    got = P.select_exits(states, bank, P.RuntimeConfig(exit_threshold=0.9)).cpu().numpy()
    assert np.all((got == want) | exc)


@pytest.mark.gpu
def test_checkpoint_capture_shape_mismatch_raises():
    need_gpu()
    routers, host, states, bank = _states_bank(64, 128, 12, [3, 7, 11], 4, torch.bfloat16,
                                               interval=4)
    head = P.OutputHead(12, 128, np.ones(128, np.float32),
                        np.ones((16, 128), np.float32))
    bad = list(states)
    bad[4] = states[4][:40]  # a shorter checkpoint capture
    with pytest.raises(ValueError, match="shape"):
        P.posthoc_select(head, bad, bank, P.RuntimeConfig(exit_threshold=0.5))
    bad = list(states)
    bad[8] = torch.zeros((64, 96), dtype=torch.bfloat16, device="cuda")  # narrower
    with pytest.raises(ValueError):
        P.select_exits(bad, bank, P.RuntimeConfig(exit_threshold=0.5))
    small = [s[:8] for s in states]
    small[12] = states[12][:6]
    with pytest.raises(ValueError):
        P.DecodeStep(small, bank, P.RuntimeConfig(exit_threshold=0.5))


@pytest.mark.gpu
def test_recorded_chain_graphs_own_their_workspace():
    """Graphs recorded for two caller streams replay concurrently: each owns
    its look-back workspace, and both give the uncached exit map."""
    need_gpu()
    from paper_2603_21365_b200 import runtime as R
    R._chain_graphs.entries.clear()
    n, d, L = 3000, 1024, 24
    ckpts = list(O.checkpoint_layers(L, 4))
    routers, host, states, bank = _states_bank(n, d, L, ckpts, 12, torch.bfloat16, scale=0.15,
                                               interval=4)
    cfg = P.RuntimeConfig(exit_threshold=0.55)
    ref = P.select_exits(states, bank, cfg)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for st in (s1, s2):
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(2):  # first call eager, second records
                P.select_exits(states, bank, cfg)
    torch.cuda.synchronize()
    recorded = [e for e in R._chain_graphs.entries.values() if e[1]]
    assert len(recorded) >= 2
    wss = {e[3][2].data_ptr() for e in recorded}
    assert len(wss) == len(recorded)
    outs = []
    for _ in range(20):
        for st in (s1, s2):
            with torch.cuda.stream(st):
                outs.append(P.select_exits(states, bank, cfg))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)


class _Block(nn.Module):
    def __init__(self, d, seed):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.lin = nn.Linear(d, d, bias=False)
        with torch.no_grad():
            self.lin.weight.copy_(torch.randn((d, d), generator=g) * (0.5 / d ** 0.5))

    def forward(self, x):
        return (x + torch.tanh(self.lin(x)),)


class _Tiny(nn.Module):
    def __init__(self, L, d):
        super().__init__()
        self.model = nn.Module()
        self.model.layers = nn.ModuleList([_Block(d, i) for i in range(L)])

    def forward(self, x):
        for layer in self.model.layers:
            x = layer(x)[0]
        return x


@pytest.mark.gpu
def test_online_hook_new_chain_per_forward():
    """Prefill then a decode step inside ONE capture context: each forward
    gets its own chain sized from its own rows (exit map of the latest
    forward, matching its post-hoc selection)."""
    need_gpu()
    from paper_2603_21365_b200.hook import CheckpointCapture
    d, L = 256, 12
    m = _Tiny(L, d).cuda().to(torch.bfloat16)
    g = np.random.Generator(np.random.PCG64(3))
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in (3, 7, 11)}
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    cfg = P.RuntimeConfig(exit_threshold=0.55)
    with torch.no_grad(), CheckpointCapture(m, bank.checkpoints, bank=bank, config=cfg,
                                            online=True) as cap:
        for rows in (2048, 24, 8, 300):
            m(torch.randn(rows, d, device="cuda").to(torch.bfloat16))
            got = cap.exit_layers
            assert got.shape == (rows,)
            want = P.select_exits(cap.hidden_states, bank, cfg)
            assert torch.equal(got, want), rows


def test_identity_cache_is_weak_and_bounded():
    """CPU: entries hit only for the same live objects, never pin them, and
    the cache is bounded."""
    c = D.IdentityCache(3)

    class Obj:
        pass

    a, arr = Obj(), np.zeros(4)
    c.put((id(a),), (a, arr), "va")
    assert c.get((id(a),), (a, arr)) == "va"
    assert c.get((id(a),), (a, np.zeros(4))) is None  # another array: miss
    c.put((id(a),), (a, arr), "va")
    del a
    gc.collect()
    b = Obj()
    assert c.get((id(b),), (b, arr)) is None
    for i in range(10):
        o = Obj()
        c.put(("k", i), (o,), i)
    assert len(c) <= 3
    P.invalidate_device_caches()
