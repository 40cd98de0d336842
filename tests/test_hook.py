"""Checkpoint-layer hook: capture indexing on CPU; online routing on GPU."""

import numpy as np
import pytest
import torch
import torch.nn as nn

import paper_2603_21365_b200 as P
from paper_2603_21365_b200.hook import CheckpointCapture, resolve_layers
from oracle import tide_oracle as O


class Block(nn.Module):
    def __init__(self, d, seed):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.lin = nn.Linear(d, d, bias=False)
        with torch.no_grad():
            self.lin.weight.copy_(torch.randn((d, d), generator=g) * (0.5 / d ** 0.5))

    def forward(self, x):
        return (x + torch.tanh(self.lin(x)),)  # HF-style tuple output


class Tiny(nn.Module):
    def __init__(self, L=12, d=64):
        super().__init__()
        self.model = nn.Module()
        self.model.layers = nn.ModuleList([Block(d, i) for i in range(L)])

    def forward(self, x):
        hs = [x]
        for layer in self.model.layers:
            x = layer(x)[0]
            hs.append(x)
        return x, hs


def test_capture_matches_full_capture():
    torch.manual_seed(0)
    m = Tiny()
    path, layers = resolve_layers(m)
    assert path == "model.layers" and len(layers) == 12
    x = torch.randn(2, 5, 64)
    with CheckpointCapture(m, (3, 7, 11)) as cap:
        _, hs = m(x)
    got = cap.hidden_states
    assert len(got) == 13
    for k in (3, 7, 11):
        assert torch.equal(got[k + 1], hs[k + 1].reshape(-1, 64))
    assert torch.equal(got[12], hs[12].reshape(-1, 64))
    assert got[0].shape == (10, 64)  # placeholder carries the width only
    assert not m.model.layers[3]._forward_hooks  # removed on exit


def test_capture_rejects_bad_checkpoint():
    with pytest.raises(ValueError):
        CheckpointCapture(Tiny(), (3, 12))


@pytest.mark.gpu
def test_online_routing_equals_posthoc():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d, L = 256, 12
    m = Tiny(L, d).cuda().to(torch.bfloat16)
    g = np.random.Generator(np.random.PCG64(3))
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in (3, 7, 11)}
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    cfg = P.RuntimeConfig(exit_threshold=0.55)
    x = torch.randn(8, 512, d, device="cuda").to(torch.bfloat16)
    with torch.no_grad(), CheckpointCapture(m, bank.checkpoints, bank=bank, config=cfg,
                                            online=True) as cap:
        m(x)
    online = cap.exit_layers.cpu().numpy()
    offline = P.select_exits(cap.hidden_states, bank, cfg).cpu().numpy()
    np.testing.assert_array_equal(online, offline)
    assert (online >= 0).any() and (online < 0).any()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,shape", [(torch.bfloat16, (8, 512)), (torch.float16, (3, 700)),
                                         (torch.bfloat16, (8, 1)), (torch.float32, (4, 300))])
def test_online_routing_matches_oracle(dtype, shape):
    """Online routing inside the layer hooks (link per checkpoint as the
    forward runs; decode-sized batches too) == the oracle's first-exit map of
    the captured checkpoint rows (ee/runtime.py:151-178 per-token, band rule of
    SURVEY.md §8c) — the oracle, not the CUDA path, is the reference here."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from tests.gpu_helpers import RTOL
    d, L = 256, 12
    m = Tiny(L, d).cuda().to(dtype)
    g = np.random.Generator(np.random.PCG64(5))
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in (3, 7, 11)}
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    theta = 0.55
    cfg = P.RuntimeConfig(exit_threshold=theta)
    x = torch.randn(*shape, d, device="cuda").to(dtype)
    with torch.no_grad(), CheckpointCapture(m, bank.checkpoints, bank=bank, config=cfg,
                                            online=True) as cap:
        m(x)
    got = cap.exit_layers.cpu().numpy()
    hs = cap.hidden_states
    scores, exc = {}, np.zeros(got.shape[0], bool)
    tol = RTOL["f32" if dtype == torch.float32 else "bf16"]
    for k, r in routers.items():
        s, t, mm = O.route_logits(hs[k + 1].float().cpu().numpy(), r)
        scores[k] = s
        exc |= np.abs(t - O.logit_of(theta)) <= tol * np.maximum(np.abs(t), mm)
    want = O.first_exit_from_scores(scores, theta)
    assert np.all((got == want) | exc), int(((got != want) & ~exc).sum())
    assert exc.mean() < 0.5  # the band does not excuse everything
