"""GPU parity: calibration labeller (compute_labels / batched_cosine_similarity)
vs the reference golden vectors — restates pkg/tests/test_calibration.py:138-193
and test_tensor_math.py:123-170 against the kernel."""

import numpy as np
import pytest
import torch

import paper_2603_21365_b200 as P
from oracle import tide_oracle as O
from tests.golden.cases import LABEL_CASES, digest, make_label_inputs, stored_digest
from tests.gpu_helpers import need_gpu, to_dev

pytestmark = pytest.mark.gpu


def _states(ckpts, final):
    return P.CollectedStates(checkpoint_states=ckpts, final_states=final,
                             token_count=len(final), corpus_digest="t")


@pytest.mark.parametrize("name", sorted(LABEL_CASES))
def test_labels_match_golden(golden_labels, name):
    need_gpu()
    spec = LABEL_CASES[name]
    ckpts, final = make_label_inputs(spec)
    assert digest(final, *[ckpts[k] for k in sorted(ckpts)]) == stored_digest(
        golden_labels, f"{name}__digest")
    dt = spec["dtype"]
    if dt == "f32":
        ds = P.compute_labels(_states(ckpts, final), spec["tau"])
        get = lambda x: x  # noqa: E731
    else:
        dev_ck = {k: to_dev(v, dt) for k, v in ckpts.items()}
        ds = P.compute_labels(_states(dev_ck, to_dev(final, dt)), spec["tau"])
        get = lambda x: x.cpu().numpy()  # noqa: E731
    assert ds.zero_norm_count == int(golden_labels[f"{name}__zero"][0])
    for k in sorted(ckpts):
        ws = golden_labels[f"{name}__sims_{k}"]
        np.testing.assert_allclose(get(ds.similarities[k]), ws, atol=1e-6, rtol=0)
        wl = golden_labels[f"{name}__labels_{k}"]
        near = np.abs(ws - np.float32(spec["tau"])) <= 1e-6
        got = get(ds.labels[k])
        assert got.dtype == np.float32
        assert np.all((got == wl) | near)


def test_reference_label_properties(rng):
    need_gpu()
    h = rng.standard_normal((20, 8), dtype=np.float32)
    assert np.all(P.compute_labels(_states({3: h.copy()}, h.copy()), 0.98).labels[3] == 1.0)
    assert np.all(P.compute_labels(_states({3: h.copy()}, -h), 0.98).labels[3] == 0.0)
    h = rng.standard_normal((5, 8), dtype=np.float32)
    final = h.copy()
    h[1] = 0.0
    final[3] = 0.0
    ds = P.compute_labels(_states({3: h}, final), 0.5)
    assert ds.zero_norm_count == 2
    assert ds.labels[3][1] == 0.0 and ds.labels[3][3] == 0.0 and ds.similarities[3][1] == 0.0
    h = rng.standard_normal((50, 16), dtype=np.float32)
    f = h + rng.standard_normal((50, 16), dtype=np.float32) * 0.2
    low = P.compute_labels(_states({3: h}, f), 0.9).labels[3]
    high = P.compute_labels(_states({3: h}, f), 0.99).labels[3]
    assert np.all(high <= low)
    with pytest.raises(ValueError):
        P.compute_labels(_states({3: h}, h), 1.0)


def test_batched_cosine_matches_oracle(rng):
    need_gpu()
    a = rng.standard_normal((40, 16), dtype=np.float32)
    b = rng.standard_normal((40, 16), dtype=np.float32)
    sims, zero = P.batched_cosine_similarity(a, b)
    ws, wz = O.batched_cosine_similarity(a, b)
    np.testing.assert_allclose(sims, ws, atol=1e-6)
    assert not zero.any()
    a[2] = 0.0
    sims, zero = P.batched_cosine_similarity(a, b)
    assert zero.tolist() == [i == 2 for i in range(40)] and sims[2] == 0.0
    for s in range(10):
        g = np.random.Generator(np.random.PCG64(s))
        x = (g.standard_normal((8, 12)) * 10.0 ** float(g.integers(-3, 4))).astype(np.float32)
        y = (g.standard_normal((8, 12)) * 10.0 ** float(g.integers(-3, 4))).astype(np.float32)
        sm, _ = P.batched_cosine_similarity(x, y)
        assert np.all(sm >= -1.0) and np.all(sm <= 1.0)


def test_labeller_large_bf16_vs_oracle():
    """Config-4 shape slice: d=4096, 8 checkpoints + final, bf16, on device."""
    need_gpu()
    n, d, C = 20000, 4096, 8
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    fin = torch.randn((n, d), generator=gen, device="cuda").to(torch.bfloat16)
    cks = {3 + 4 * i: (fin.float() + 0.15 * (1 + 0.25 * i) *
                       torch.randn((n, d), generator=gen, device="cuda")).to(torch.bfloat16)
           for i in range(C)}
    layers, sims, labels, zero = P.label_tensors(cks, fin, 0.98, labels_dtype="u8")
    f = fin.float().cpu().numpy()
    for i, k in enumerate(layers):
        if i % 3:
            continue
        ws, wz = O.batched_cosine_similarity(cks[k].float().cpu().numpy(), f)
        np.testing.assert_allclose(sims[i].cpu().numpy(), ws, atol=2e-6)
        wl = ws > np.float32(0.98)
        got = labels[i].cpu().numpy().astype(bool)
        near = np.abs(ws - np.float32(0.98)) <= 2e-6
        assert np.all((got == wl) | near)
    assert int(zero.sum()) == 0
