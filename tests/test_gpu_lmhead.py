"""GPU parity of the tensor-core LM head (tide_lm_head, csrc/lmhead.cu) and the
bf16-pair staging (tide_select_project_split) against the oracle's
lm_head_from_hidden (ee/model.py:329-338) and an f64 product of the same
operands.

Tolerance: with A, B given as bf16 pairs (x = hi + lo to
2^-17 relative) and the three MMA terms hi.hi + hi.lo + lo.hi accumulated in
f32, |logit - exact| <= 1e-5 * M, M = sum_j |a_j b_j| (the conditioning
magnitude of the dot product, as for the router logits); the hi-only form
(bf16 products) is held to 1e-2 * M."""

import numpy as np
import pytest
import torch

import paper_2603_21365_b200 as P
from oracle import tide_oracle as O
from tests.gpu_helpers import need_gpu

pytestmark = pytest.mark.gpu


FORMS = ["persistent", "pair", "one"]


def _set_form(monkeypatch, form):
    """persistent CTA pairs (the default for 3 terms), one-tile CTA pairs, one CTA."""
    monkeypatch.setenv("TIDE_LM_PAIR", "0" if form == "one" else "1")
    monkeypatch.setenv("TIDE_LM_PERSIST", "1" if form == "persistent" else "0")


def _lm(a32, b32, terms, ldo=None, extra_rows=0, full=False):
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N
    from paper_2603_21365_b200.runtime import split_bf16

    dev = torch.device("cuda", 0)
    n, d = a32.shape
    V = b32.shape[0]
    ld = (d + 7) // 8 * 8
    ah, al = split_bf16(torch.from_numpy(a32).to(dev), ld)
    bh, bl = split_bf16(torch.from_numpy(b32).to(dev), ld)
    ldo = (V + 3) // 4 * 4 if ldo is None else ldo
    out = torch.full((n + extra_rows, ldo), float("nan"), dtype=torch.float32, device=dev)
    rc = N.load().tide_lm_head(ah.data_ptr(), al.data_ptr() if terms == 3 else None, ld, n, d,
                               bh.data_ptr(), bl.data_ptr() if terms == 3 else None, ld, V,
                               out.data_ptr(), ldo, Dv.stream_handle(dev))
    N.check(rc, "tide_lm_head")
    torch.cuda.synchronize()
    return out.cpu().numpy() if full else out[:n, :V].cpu().numpy()


@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("n,d,V", [(1, 64, 64), (8, 4096, 1000), (130, 772, 300),
                                   (1000, 1024, 2500), (300, 4096, 50257), (129, 256, 129)])
def test_lm_head_three_terms_f32_grade(n, d, V, form, monkeypatch):
    """Every form: persistent CTA pairs (cta_group::2, the default for 3
    terms; ragged row counts leave the pair's second CTA partly or wholly
    past the rows), one-tile CTA pairs and the one-CTA kernel."""
    need_gpu()
    _set_form(monkeypatch, form)
    g = np.random.Generator(np.random.PCG64(n + d + V))
    a = g.standard_normal((n, d), dtype=np.float32)
    b = (g.standard_normal((V, d)) * 0.02).astype(np.float32)
    got = _lm(a, b, 3)
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    M = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
    err = np.abs(got - exact) / M
    assert np.isfinite(got).all()
    assert err.max() <= 1e-5, err.max()
    # and as close to numpy's own f32 GEMM as numpy is to the exact product
    f32 = a @ b.T
    assert np.abs(got - f32).max() <= 4 * np.abs(f32 - exact).max() + 1e-5 * M.max()


@pytest.mark.parametrize("terms", [3, 1])
@pytest.mark.parametrize("form", FORMS)
@pytest.mark.parametrize("n,d,V", [(129, 256, 129), (300, 1024, 1001), (5, 64, 32), (257, 512, 600),
                                   (2, 128, 4099)])
def test_lm_head_tma_store_epilogue(n, d, V, terms, form, monkeypatch):
    """The TMA-store epilogue (logit blocks through shared memory, clipped by
    the output tensor map) writes exactly what the per-lane stores write:
    bit-identical logits; past column V only the rest of the last 16-byte
    piece, with 0 (the C-ABI contract: columns [V, ceil4(V)) receive 0), and
    nothing past ceil4(V) (the extra padding stays NaN) or row n (the rows
    after the output stay NaN)."""
    need_gpu()
    _set_form(monkeypatch, form)
    g = np.random.Generator(np.random.PCG64(n * 7 + V))
    a = g.standard_normal((n, d), dtype=np.float32)
    b = (g.standard_normal((V, d)) * 0.02).astype(np.float32)
    v4 = (V + 3) // 4 * 4
    ldo = v4 + 8
    monkeypatch.setenv("TIDE_LM_TMA_STORE", "1")
    tma = _lm(a, b, terms, ldo=ldo, extra_rows=3, full=True)
    monkeypatch.setenv("TIDE_LM_TMA_STORE", "0")
    lane = _lm(a, b, terms, ldo=ldo, extra_rows=3, full=True)
    assert np.isfinite(tma[:n, :V]).all()
    assert np.array_equal(tma[:n, :V], lane[:n, :V])
    assert (tma[:n, V:v4] == 0).all()
    assert np.isnan(tma[:n, v4:]).all() and np.isnan(tma[n:]).all()
    assert np.isnan(lane[:n, V:]).all() and np.isnan(lane[n:]).all()


@pytest.mark.parametrize("form", FORMS)
def test_lm_head_hi_only_bf16_products(form, monkeypatch):
    need_gpu()
    _set_form(monkeypatch, form)
    g = np.random.Generator(np.random.PCG64(5))
    a = g.standard_normal((257, 512), dtype=np.float32)
    b = (g.standard_normal((600, 512)) * 0.02).astype(np.float32)
    got = _lm(a, b, 1)
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    M = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
    assert (np.abs(got - exact) / M).max() <= 1e-2


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_posthoc_logits_on_tensor_cores_match_oracle(dtype):
    """posthoc_select's logits (select_project_split + tide_lm_head) ==
    the oracle's final-norm + LM head of each row's exit layer."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(11))
    L, d, n, V = 12, 768, 500, 3000
    routers = {k: O.make_router(d, 128, k, g, scale=0.2) for k in (3, 7, 11)}
    states = [O.round_to(g.standard_normal((n, d), dtype=np.float32), dtype)
              for _ in range(L + 1)]
    fn = (1.0 + 0.1 * g.standard_normal(d)).astype(np.float32)
    lm = (g.standard_normal((V, d)) * 0.02).astype(np.float32)
    bank = P.make_bank({k: (r.w_down, r.w_up) for k, r in routers.items()}, num_layers=L)
    head = P.OutputHead(L, d, fn, lm)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    dev_states = [torch.from_numpy(s).cuda().to(tdt) for s in states]
    logits, exits = P.posthoc_select(head, dev_states, bank, P.RuntimeConfig(exit_threshold=0.6))
    e = exits.cpu().numpy()
    rows = np.stack([states[int(k) + 1][i] if k >= 0 else states[L][i] for i, k in enumerate(e)])
    want = O.lm_head_from_hidden(fn, lm, rows)
    normed = O.rmsnorm(rows, fn, O.DEFAULT_EPS).astype(np.float64)
    M = np.abs(normed) @ np.abs(lm.astype(np.float64)).T
    err = np.abs(logits.cpu().numpy() - want) / M
    assert err.max() <= 1e-5, err.max()


def test_select_project_split_is_the_f32_staging():
    """hi + lo of the split staging == the f32 staging (tide_select_project)
    to 2^-16 relative, and hi == bf16(f32 staging) exactly."""
    need_gpu()
    from paper_2603_21365_b200 import _device as Dv
    from paper_2603_21365_b200 import _native as N

    g = np.random.Generator(np.random.PCG64(3))
    n, d = 333, 1000
    x = torch.from_numpy(g.standard_normal((n, d), dtype=np.float32)).cuda()
    gain = torch.from_numpy((1 + 0.1 * g.standard_normal(d)).astype(np.float32)).cuda()
    lib = N.load()
    s = Dv.stream_handle(torch.device("cuda", 0))
    f32 = torch.empty((n, d), dtype=torch.float32, device="cuda")
    hi = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    lo = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
    ptrs = N.ptr_array([x.data_ptr()])
    N.check(lib.tide_select_project(ptrs, 1, d, N.F32, None, n, d, gain.data_ptr(), 1e-6,
                                    f32.data_ptr(), d, s), "project")
    N.check(lib.tide_select_project_split(ptrs, 1, d, N.F32, None, n, d, gain.data_ptr(), 1e-6,
                                          hi.data_ptr(), lo.data_ptr(), d, s), "split")
    torch.cuda.synchronize()
    assert torch.equal(hi, f32.to(torch.bfloat16))
    rel = ((hi.float() + lo.float()) - f32).abs() / f32.abs().clamp_min(1e-30)
    assert float(rel.max()) <= 2.0 ** -16


@pytest.mark.parametrize("terms", [3, 1])
def test_lm_head_persistent_bitwise_equals_one_tile_pairs(terms, monkeypatch):
    """The persistent pairs walk several tiles each (the ring and the
    accumulator sets carried across tiles): the same logits, bit for bit, as
    one tile per pair."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(77 + terms))
    n, d, V = 1000, 1024, 20000  # 4 row pairs x 79 vocab tiles > co-resident pairs
    a = g.standard_normal((n, d), dtype=np.float32)
    b = (g.standard_normal((V, d)) * 0.02).astype(np.float32)
    _set_form(monkeypatch, "persistent")
    got = _lm(a, b, terms)
    _set_form(monkeypatch, "pair")
    want = _lm(a, b, terms)
    assert np.isfinite(got).all()
    assert np.array_equal(got, want)
