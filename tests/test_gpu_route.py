"""GPU parity: fused RMSNorm + router + mask + compaction vs the oracle and the
reference's golden vectors (restates pkg/tests/test_router_ops.py:72-107 and
test_acceptance.py #2 against the kernels)."""

import numpy as np
import pytest
import torch

import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _device as D
from paper_2603_21365_b200 import _native as N
from oracle import tide_oracle as O
from tests.golden.cases import ROUTE_CASES, digest, make_route_inputs, stored_digest
from tests.gpu_helpers import (check_decisions, check_logits, need_gpu, to_dev)

pytestmark = pytest.mark.gpu


def _router(wd, wu, layer=3):
    return P.Router(layer=layer, w_down=wd, w_up=wu)


@pytest.mark.parametrize("name", sorted(ROUTE_CASES))
def test_route_case_matches_oracle_and_golden(golden_route, name):
    need_gpu()
    spec = ROUTE_CASES[name]
    h, wd, wu = make_route_inputs(spec)
    assert digest(h, wd, wu) == stored_digest(golden_route, f"{name}__digest")
    router = _router(wd, wu)
    oref = O.OracleRouter(3, wd, wu)
    s_ref, t_ref, m_ref = O.route_logits(h, oref)
    dt = spec["dtype"]
    x = to_dev(h, dt)
    r = P.route(x, router, theta=0.5, want_logits=True, want_indices=True)
    scores = r["scores"].cpu().numpy()
    logits = r["logits"].cpu().numpy()
    check_logits(logits, t_ref, m_ref, dt, name)
    # scores are sigma(logit) in f64 -> f32, bounded in [0, 1]
    assert np.all(scores >= 0) and np.all(scores <= 1)
    np.testing.assert_array_equal(scores, np.array([O._sigma64(float(v)) for v in logits],
                                                   np.float32))
    if dt == "f32":
        # reference criterion #2 (test_acceptance.py:70-87): within 1e-5 of the reference
        assert np.max(np.abs(scores - golden_route[f"{name}__fused"])) <= 1e-5
    mask = r["mask"].cpu().numpy()
    check_decisions(mask, t_ref, m_ref, 0.5, dt, name)
    # compaction is bit-exact against the oracle applied to the GPU's own mask
    e, c = O.compact_indices(mask)
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)
    if spec["kind"] == "rigged":
        zero = set(spec.get("zero_rows", ()))
        for i in range(spec["n"]):
            want = 0.5 if i in zero else (1.0 if spec["hot"] else 0.0)
            assert scores[i] == want, (i, scores[i], want)


@pytest.mark.parametrize("name", sorted(ROUTE_CASES))
def test_route_scores_matches_reference_composed(golden_route, name):
    """route_scores (the composed equivalence partner, ee/router_ops.py:60-65)
    on the device against the REFERENCE's own composed scores recorded in
    the golden fixture (not against the fused kernel): within 1e-5 (f32
    products) for f32 inputs, the bf16 band for bf16 / f16 captures."""
    need_gpu()
    key = f"{name}__composed"
    if key not in golden_route.files:
        pytest.skip("no composed vector recorded for this case")
    spec = ROUTE_CASES[name]
    h, wd, wu = make_route_inputs(spec)
    want = golden_route[key]
    got = P.route_scores(to_dev(h, spec["dtype"]), _router(wd, wu))
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    tol = 1e-5 if spec["dtype"] == "f32" else 2e-2
    assert got.shape == want.shape
    assert np.max(np.abs(got.astype(np.float64) - want)) <= tol


@pytest.mark.parametrize("theta", [1.0, 0.85, 0.5, 0.1])
def test_threshold_rule_and_off_switch(theta):
    need_gpu()
    h, wd, wu = make_route_inputs(ROUTE_CASES["bf16_4096x128"])
    router = _router(wd, wu)
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "bf16"), router, theta=theta, want_indices=True)
    mask = r["mask"].cpu().numpy()
    check_decisions(mask, t_ref, m_ref, theta, "bf16", f"theta={theta}")
    if theta == 1.0:
        assert not mask.any()
        assert r["exiting_indices"].numel() == 0


def test_host_api_matches_reference_semantics(rng):
    """pkg/tests/test_router_ops.py:72-107 restated on the kernels (host numpy API)."""
    need_gpu()
    router = P.Router(layer=3, w_down=rng.standard_normal((32, 64), dtype=np.float32),
                      w_up=rng.standard_normal((1, 32), dtype=np.float32))
    h = rng.standard_normal((200, 64), dtype=np.float32) * 5
    fused = P.fused_layernorm_route(h, router)
    assert isinstance(fused, np.ndarray) and fused.dtype == np.float32
    composed = P.route_scores(h, router)
    assert np.max(np.abs(fused - composed)) <= 1e-5
    big = P.fused_layernorm_route(h * 100, router)
    assert np.all(big >= 0.0) and np.all(big <= 1.0)
    assert P.fused_layernorm_route(np.zeros((1, 64), np.float32), router)[0] == 0.5
    a = P.fused_layernorm_route(h[:10], router)
    b = P.fused_layernorm_route(h[:10] * 1000.0, router)
    np.testing.assert_allclose(a, b, atol=1e-5)
    with pytest.raises(ValueError, match="expected"):
        P.fused_layernorm_route(np.zeros((3, 32), np.float32), router)
    assert P.fused_layernorm_route(np.zeros((0, 64), np.float32), router).shape == (0,)


def test_tensor_core_path_selected():
    need_gpu()
    lib = N.load()
    assert lib.tide_route_uses_tensor_cores(N.BF16, 4096, 128) == 1
    assert lib.tide_route_uses_tensor_cores(N.F16, 8192, 256) == 1
    assert lib.tide_route_uses_tensor_cores(N.F32, 4096, 128) == 1   # 3xTF32, >= 16,384 rows
    assert lib.tide_route_uses_tensor_cores(N.F32, 16384, 128) == 0  # outside its 1e-5 range


@pytest.fixture(params=["split", "persistent"])
def k1_mode(request, monkeypatch):
    """Small row counts take the split-K cluster kernel unless TIDE_SPLIT=0."""
    if request.param == "persistent":
        monkeypatch.setenv("TIDE_SPLIT", "0")
    else:
        monkeypatch.delenv("TIDE_SPLIT", raising=False)
    return request.param


@pytest.mark.parametrize("n", [1, 31, 32, 33, 127, 128, 129, 500, 4099, 9500, 20000])
def test_ragged_sizes_bf16(n, k1_mode):
    """Every tile / group boundary: 32-row boxes, partial tiles, multi-group CTAs."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(1000 + n))
    d, b = 512, 128
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.05).astype(np.float32)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "bf16"), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "bf16", f"n={n}")
    mask = r["mask"].cpu().numpy()
    e, c = O.compact_indices(mask)
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


def test_gathered_rows_equal_dense_on_subset(k1_mode):
    """row_idx (peeling) mode == dense route over h[row_idx]; ids mapped back."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(77))
    n, d, b = 3000, 1024, 128
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.05).astype(np.float32)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
    x = to_dev(h, "bf16")
    router = _router(wd, wu)
    sub = np.sort(g.choice(n, size=1777, replace=False)).astype(np.int64)
    wdd, wud = P.router_ops.device_weights(router, N.BF16, x.device)
    m = len(sub)
    idx = torch.from_numpy(sub).cuda()
    logits = torch.empty(m, dtype=torch.float32, device="cuda")
    mask = torch.empty(m, dtype=torch.uint8, device="cuda")
    cont = torch.empty(m, dtype=torch.int64, device="cuda")
    ex = torch.empty(m, dtype=torch.int64, device="cuda")
    counts = torch.empty(2, dtype=torch.int64, device="cuda")
    exit_layers = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    lib = N.load()
    N.check(lib.tide_route(x.data_ptr(), d, m, None, n, d, N.BF16, idx.data_ptr(),
                           wdd.data_ptr(), wud.data_ptr(), b, 1e-6, 0.5, 9, None,
                           logits.data_ptr(), mask.data_ptr(), ex.data_ptr(), cont.data_ptr(), 1,
                           exit_layers.data_ptr(), counts.data_ptr(),
                           D.workspace().data_ptr(), D.stream_handle()), "tide_route")
    dense = P.route(x[idx], router, theta=0.5, want_logits=True)
    np.testing.assert_array_equal(logits.cpu().numpy(), dense["logits"].cpu().numpy())
    mk = mask.cpu().numpy().astype(bool)
    ne = int(counts[0])
    assert ne == mk.sum() and int(counts[1]) == m - ne
    np.testing.assert_array_equal(ex.cpu().numpy()[:ne], sub[mk])
    np.testing.assert_array_equal(cont.cpu().numpy()[: m - ne], sub[~mk])
    el = exit_layers.cpu().numpy()
    assert np.all(el[sub[mk]] == 9) and np.all(el[np.setdiff1d(np.arange(n), sub[mk])] == -1)


def test_device_count_input(k1_mode):
    """n read from device memory (the peeling chain's counts[1])."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(78))
    n, d, b = 1000, 256, 64
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.05).astype(np.float32)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
    x = to_dev(h, "bf16")
    router = _router(wd, wu)
    wdd, wud = P.router_ops.device_weights(router, N.BF16, x.device)
    for live in (0, 1, 37, 640, 1000):
        ndev = torch.tensor([0, live], dtype=torch.int64, device="cuda")
        logits = torch.full((n,), 7.0, dtype=torch.float32, device="cuda")
        counts = torch.full((2,), -5, dtype=torch.int64, device="cuda")
        N.check(N.load().tide_route(x.data_ptr(), d, n, ndev.data_ptr() + 8, n, d, N.BF16, None,
                                    wdd.data_ptr(), wud.data_ptr(), b, 1e-6, 0.5, 1, None,
                                    logits.data_ptr(), None, None, None, 0, None,
                                    counts.data_ptr(), D.workspace().data_ptr(),
                                    D.stream_handle()), "tide_route")
        lg = logits.cpu().numpy()
        assert np.all(lg[live:] == 7.0)
        if live:
            ref = P.route(x[:live], router, want_logits=True)["logits"].cpu().numpy()
            np.testing.assert_array_equal(lg[:live], ref)
        assert int(counts[0]) + int(counts[1]) == live


def test_repeated_launches_reuse_workspace():
    """The epoch-tagged look-back state needs no reset between launches."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(79))
    n, d, b = 9000, 256, 128
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.05).astype(np.float32)
    router = _router(wd, wu)
    for it in range(6):
        h = O.round_to(g.standard_normal((n, d), dtype=np.float32), "bf16")
        r = P.route(to_dev(h, "bf16"), router, theta=0.5, want_indices=True)
        e, c = O.compact_indices(r["mask"].cpu().numpy())
        np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
        np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


@pytest.mark.parametrize("d,b,n", [(200, 40, 700), (1000, 96, 3000), (4096, 128, 4096),
                                   (8192, 16, 1500), (8192, 128, 8192), (512, 256, 300)])
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_split_and_persistent_agree_with_oracle(d, b, n, dtype, monkeypatch):
    """Both K1 variants (split-K cluster / persistent) against the oracle, incl.
    widths that are not multiples of 64 and bottlenecks that are not of 32."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(d * 7 + b + n))
    wd = (g.standard_normal((b, d)) * (1.0 / np.sqrt(d))).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32), dtype)
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("TIDE_SPLIT", mode)
        r = P.route(to_dev(h, dtype), _router(wd, wu), theta=0.5, want_logits=True,
                    want_indices=True)
        check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, dtype, f"split={mode}")
        e, c = O.compact_indices(r["mask"].cpu().numpy())
        np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
        np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)
        out[mode] = r["logits"].cpu().numpy()
    np.testing.assert_allclose(out["1"], out["0"], rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("n,gathered", [(100_000, False), (160_000, False), (90_000, True)])
def test_multi_group_persistent_ctas(n, gathered):
    """More rows than one group per SM (148 x 512): CTAs loop over several
    groups (accumulator reuse, ring phases carried across groups, epilogue of
    group g overlapping group g+1's first chunks)."""
    need_gpu()
    import torch
    g = np.random.Generator(np.random.PCG64(4242 + n))
    d, b = 256, 128
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.05).astype(np.float32)
    rows = 2 * n if gathered else n
    h = O.round_to(g.standard_normal((rows, d), dtype=np.float32), "bf16")
    hd = to_dev(h, "bf16")
    router = _router(wd, wu)
    if gathered:
        idx = np.sort(g.choice(rows, size=n, replace=False)).astype(np.int64)
        wdd, wud = P.router_ops.device_weights(router, N.BF16, hd.device)
        it = torch.from_numpy(idx).cuda()
        r = {k: torch.empty(n, dtype=t, device="cuda") for k, t in
             (("logits", torch.float32), ("mask", torch.uint8), ("exiting_indices", torch.int64),
              ("continuing_indices", torch.int64))}
        counts = torch.empty(2, dtype=torch.int64, device="cuda")
        N.check(N.load().tide_route(hd.data_ptr(), d, n, None, rows, d, N.BF16, it.data_ptr(),
                                    wdd.data_ptr(), wud.data_ptr(), b, 1e-6, 0.5, 9, None,
                                    r["logits"].data_ptr(), r["mask"].data_ptr(),
                                    r["exiting_indices"].data_ptr(),
                                    r["continuing_indices"].data_ptr(), 0, None,
                                    counts.data_ptr(), D.workspace().data_ptr(),
                                    D.stream_handle()), "tide_route")
        ne = int(counts[0])
        r["exiting_indices"] = r["exiting_indices"][:ne]
        r["continuing_indices"] = r["continuing_indices"][: n - ne]
        hsel = h[idx]
    else:
        r = P.route(hd, router, theta=0.5, want_logits=True, want_indices=True)
        hsel = h
    _, t_ref, m_ref = O.route_logits(hsel, O.OracleRouter(3, wd, wu))
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "bf16", f"n={n}")
    mask = r["mask"].cpu().numpy()
    assert O.decision_band_ok(mask, t_ref, m_ref, 0.5, 2e-2).all()
    e, c = O.compact_indices(mask)
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


def test_headline_shape_full_size():
    """The bench workload itself: 65,536 x 4096 bf16, one checkpoint.  Logits
    on a 4,096-row sample; every decision by the band rule; compaction exact."""
    need_gpu()
    import torch
    g = np.random.Generator(np.random.PCG64(202))
    orouter = O.make_router(4096, 128, 3, g)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234)
    hd = torch.randn((65536, 4096), generator=gen, device="cuda").to(torch.bfloat16)
    r = P.route(hd, P.Router(3, orouter.w_down, orouter.w_up), theta=0.5, want_logits=True,
                want_indices=True)
    h = hd.float().cpu().numpy()
    _, t_ref, m_ref = O.route_logits(h, orouter)
    logits = r["logits"].cpu().numpy()
    check_logits(logits[:4096], t_ref[:4096], m_ref[:4096], "bf16", "headline sample")
    mask = r["mask"].cpu().numpy()
    assert O.decision_band_ok(mask, t_ref, m_ref, 0.5, 2e-2).all()
    e, c = O.compact_indices(mask)
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


@pytest.mark.parametrize("n,d", [(20000, 256), (70000, 128)])
def test_f32_many_blocks_with_compaction(n, d):
    """CUDA-core f32 kernel with more 16-row blocks than co-resident CTAs and
    the look-back on (regression: a grid larger than what fits on the SMs
    deadlocked the look-back)."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(n + d))
    b = 128
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = g.standard_normal((n, d), dtype=np.float32)
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "f32"), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "f32", f"n={n}")
    e, c = O.compact_indices(r["mask"].cpu().numpy())
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


@pytest.mark.parametrize("n,d,b", [(2048, 768, 128), (1000, 772, 96), (300, 100, 40),
                                   (9000, 256, 128)])
def test_f32_tensor_core_opt_in(n, d, b, monkeypatch):
    """Opt-in 3xTF32 tcgen05 kernel (TIDE_F32_TC=1, route_tf32.cu) inside the
    f32 contract at GPT-2-small widths; compaction bit-exact."""
    need_gpu()
    monkeypatch.setenv("TIDE_F32_TC", "1")
    assert N.load().tide_route_uses_tensor_cores(N.F32, d, b) == 1
    g = np.random.Generator(np.random.PCG64(3 * n + d + b))
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = g.standard_normal((n, d), dtype=np.float32) * 3.0
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "f32"), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "f32", f"tf32 n={n} d={d}")
    e, c = O.compact_indices(r["mask"].cpu().numpy())
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


@pytest.mark.parametrize("n,d,b", [(20000, 4096, 128), (16384, 8192, 128), (65536, 4096, 128),
                                   (30000, 1000, 96)])
def test_f32_default_tensor_cores_within_contract(n, d, b):
    """f32 rows from 16,384 on take the 3xTF32 tcgen05 kernel by default
    (segmented TMEM accumulators): logits inside the 1e-5 f32 contract at
    d <= 8192, compaction bit-exact."""
    need_gpu()
    assert N.load().tide_route_uses_tensor_cores(N.F32, d, b) == 1
    g = np.random.Generator(np.random.PCG64(7 * n + d))
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = g.standard_normal((n, d), dtype=np.float32) * 3.0
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "f32"), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "f32", f"tf32 default n={n} d={d}")
    e, c = O.compact_indices(r["mask"].cpu().numpy())
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


@pytest.mark.parametrize("acc", ["2", "4"])
def test_f32_tensor_core_accumulator_layouts(acc, monkeypatch):
    """The segmented TMEM accumulator layouts (2 / 4 per tile) are inside the
    f32 contract at d = 2048 (one accumulator is not: 1.06e-5 there) with a
    bit-exact compaction."""
    need_gpu()
    monkeypatch.setenv("TIDE_F32_TC", "1")
    monkeypatch.setenv("TIDE_TF32_ACC", acc)
    n, d, b = 5000, 2048, 128
    g = np.random.Generator(np.random.PCG64(99))
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = g.standard_normal((n, d), dtype=np.float32) * 3.0
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "f32"), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "f32", f"tf32 acc={acc}")
    e, _ = O.compact_indices(r["mask"].cpu().numpy())
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)


@pytest.mark.parametrize("dtype,n,d,b", [("f32", 9000, 768, 128), ("f32", 7200, 100, 40),
                                         ("bf16", 8000, 512, 300)])
def test_wide_cuda_core_kernel(dtype, n, d, b):
    """64-row CUDA-core kernel (n above its threshold): f32 rows, a ragged
    width / bottleneck, and a bf16 shape the tensor-core kernel does not take
    (b > 256); compaction bit-exact."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(n + d + b))
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = O.round_to(g.standard_normal((n, d), dtype=np.float32), dtype)
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, dtype), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, dtype, f"wide n={n}")
    e, c = O.compact_indices(r["mask"].cpu().numpy())
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
    np.testing.assert_array_equal(r["continuing_indices"].cpu().numpy(), c)


@pytest.mark.parametrize("pair", ["1", "0"])
def test_repeated_launches_bitwise_identical(pair, monkeypatch):
    """Several row groups per CTA (160,000 rows): repeated launches, each after
    an L2-thrashing write, give bit-identical logits / masks / indices (fixed
    reduction orders).  Regression for the slot-release races found by
    tools/stress_k1.py (owner-only releases, release before the smem reads
    were consumed)."""
    need_gpu()
    import torch
    monkeypatch.setenv("TIDE_K1_PAIRSLOT", pair)
    g = np.random.Generator(np.random.PCG64(77))
    d = 2048
    wd = (g.standard_normal((128, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, 128)) * 0.05).astype(np.float32)
    router = _router(wd, wu)
    h = torch.randn((160_000, d), device="cuda").to(torch.bfloat16)
    junk = torch.empty(1 << 26, device="cuda")
    kw = dict(theta=0.5, want_logits=True, want_mask=True, want_indices=True)
    ref = P.route(h, router, **kw)
    for i in range(25):
        junk.fill_(float(i))
        r = P.route(h, router, **kw)
        for k in ("logits", "mask", "exiting_indices", "continuing_indices"):
            assert torch.equal(r[k], ref[k]), (i, k)


@pytest.mark.parametrize("b", [16, 48, 64, 96, 112, 128])
@pytest.mark.parametrize("n,d", [(20000, 1024), (3000, 4096)])
def test_f32_tensor_core_ring_shapes_bitwise(n, d, b, monkeypatch):
    """The 3xTF32 kernel's default ring (up to 4 W slots, route_tf32.cu), the
    two-W-slot ring, and W split in the kernel instead of by the pre-split
    kernel give bit-identical logits, masks and indices (they reorder waits,
    never arithmetic), over bottleneck widths whose rings differ in every
    slot count."""
    need_gpu()
    monkeypatch.setenv("TIDE_F32_TC", "1")
    g = np.random.Generator(np.random.PCG64(n + d + b))
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = to_dev(g.standard_normal((n, d), dtype=np.float32) * 3.0, "f32")
    outs = []
    for ring, presplit in ((None, "1"), ("2,0,0", "1"), ("2,0,0", "0")):
        monkeypatch.setenv("TIDE_TF32_PRESPLIT", presplit)
        if ring:
            monkeypatch.setenv("TIDE_TF32_RING", ring)
        r = P.route(h, _router(wd, wu), theta=0.5, want_logits=True, want_indices=True)
        outs.append({k: r[k].cpu().numpy() for k in ("logits", "mask", "exiting_indices",
                                                       "continuing_indices")})
    for o in outs[1:]:
        for k in outs[0]:
            np.testing.assert_array_equal(outs[0][k], o[k], err_msg=k)
    if d <= 1024:  # inside the default path's (d, b) range: the 1e-5 contract too
        _, t_ref, m_ref = O.route_logits(h.cpu().numpy(), O.OracleRouter(3, wd, wu))
        check_logits(outs[0]["logits"], t_ref, m_ref, "f32", f"ring b={b}")


@pytest.mark.parametrize("d,b", [(2048, 32), (4096, 64), (4096, 96), (1024, 16)])
def test_f32_default_narrow_bottlenecks_within_contract(d, b):
    """Narrow bottlenecks at the widest d the default 3xTF32 path takes for
    them (4 TMEM accumulators): inside the 1e-5 f32 contract."""
    need_gpu()
    n = 16384
    assert N.load().tide_route_uses_tensor_cores(N.F32, d, b) == 1
    g = np.random.Generator(np.random.PCG64(d * b))
    wd = (g.standard_normal((b, d)) * 0.05).astype(np.float32)
    wu = (g.standard_normal((1, b)) * 0.3).astype(np.float32)
    h = g.standard_normal((n, d), dtype=np.float32) * 3.0
    _, t_ref, m_ref = O.route_logits(h, O.OracleRouter(3, wd, wu))
    r = P.route(to_dev(h, "f32"), _router(wd, wu), theta=0.5, want_logits=True,
                want_indices=True)
    check_logits(r["logits"].cpu().numpy(), t_ref, m_ref, "f32", f"tf32 narrow d={d} b={b}")
    e, c = O.compact_indices(r["mask"].cpu().numpy())
    np.testing.assert_array_equal(r["exiting_indices"].cpu().numpy(), e)
