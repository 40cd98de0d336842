"""GPU parity: standalone stable compaction (batch_compact) and exit
scatter / projection — restates pkg/tests/test_router_ops.py:109-231 and
test_acceptance.py #7 against the kernels; bit-exact vs the reference."""

import numpy as np
import pytest
import torch

import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _device as D
from paper_2603_21365_b200 import _native as N
from oracle import tide_oracle as O
from tests.gpu_helpers import need_gpu

pytestmark = pytest.mark.gpu


def naive_partition(mask):
    cont = [i for i in range(len(mask)) if not mask[i]]
    exi = [i for i in range(len(mask)) if mask[i]]
    return cont, exi


def test_golden_masks_bit_exact(golden_compact):
    need_gpu()
    g = golden_compact
    for i in range(int(g["n_masks"][0])):
        mask = g[f"m{i}__mask"]
        h = np.arange(mask.shape[0] * 3, dtype=np.float32).reshape(-1, 3)
        for strategy in ("small", "prefix", "auto"):
            r = P.batch_compact(h, mask, strategy=strategy)
            key = "small" if strategy == "small" else "prefix"
            np.testing.assert_array_equal(r.exiting_indices, g[f"m{i}__{key}__exit"])
            np.testing.assert_array_equal(r.continuing_indices, g[f"m{i}__{key}__cont"])
            np.testing.assert_array_equal(r.exiting, h[r.exiting_indices])
            np.testing.assert_array_equal(r.continuing, h[r.continuing_indices])


def test_acceptance_7_exhaustive_and_random():
    """test_acceptance.py:167-210: all 256 masks at batch 8, 200 random at 1000."""
    need_gpu()
    rng = np.random.Generator(np.random.PCG64(707))
    rows8 = rng.standard_normal((8, 5), dtype=np.float32)
    for bits in range(256):
        mask = np.array([(bits >> i) & 1 == 1 for i in range(8)])
        r = P.batch_compact(rows8, mask)
        c, e = naive_partition(mask)
        np.testing.assert_array_equal(r.exiting_indices, e)
        np.testing.assert_array_equal(r.continuing_indices, c)
        rebuilt = np.zeros_like(rows8)
        rebuilt[np.asarray(c, np.int64)] = r.continuing
        P.exit_scatter(r.exiting, r.exiting_indices, rebuilt)
        np.testing.assert_array_equal(rebuilt, rows8)
    rows = torch.from_numpy(rng.standard_normal((1000, 7), dtype=np.float32)).cuda()
    for _ in range(200):
        mask = rng.random(1000) < rng.random()
        r = P.batch_compact(rows, torch.from_numpy(mask).cuda())
        c, e = naive_partition(mask)
        np.testing.assert_array_equal(r.exiting_indices.cpu().numpy(), e)
        np.testing.assert_array_equal(r.continuing_indices.cpu().numpy(), c)
        np.testing.assert_array_equal(r.exiting.cpu().numpy(), rows.cpu().numpy()[e])


@pytest.mark.parametrize("n", [0, 1, 2047, 2048, 2049, 100_000, 1_000_003])
def test_large_and_ragged_masks(n):
    need_gpu()
    g = np.random.Generator(np.random.PCG64(n + 5))
    mask = g.random(n) < 0.37
    dm = torch.from_numpy(mask.astype(np.uint8)).cuda()
    ex = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    co = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    counts = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    N.check(N.load().tide_compact(dm.data_ptr() if n else 0, n, None, None, 0, None, 0, 0, 0,
                                  ex.data_ptr(), co.data_ptr(), None, None, counts.data_ptr(),
                                  D.workspace().data_ptr(), D.stream_handle()), "tide_compact")
    e, c = O.compact_indices(mask)
    assert int(counts[0]) == len(e) and int(counts[1]) == len(c)
    np.testing.assert_array_equal(ex[: len(e)].cpu().numpy(), e)
    np.testing.assert_array_equal(co[: len(c)].cpu().numpy(), c)


def test_all_and_none_exit(rng):
    need_gpu()
    h = rng.standard_normal((9, 4), dtype=np.float32)
    all_out = P.batch_compact(h, np.ones(9, bool))
    assert all_out.continuing.shape == (0, 4)
    np.testing.assert_array_equal(all_out.exiting, h)
    none_out = P.batch_compact(h, np.zeros(9, bool))
    assert none_out.exiting.shape == (0, 4)
    np.testing.assert_array_equal(none_out.continuing, h)


def test_compact_errors_match_reference():
    need_gpu()
    with pytest.raises(ValueError, match="mask"):
        P.batch_compact(np.zeros((4, 2), np.float32), np.zeros(3, bool))
    with pytest.raises(ValueError, match="strategy"):
        P.batch_compact(np.zeros((2, 2), np.float32), np.zeros(2, bool), strategy="warp")


def test_bf16_rows_gather_bit_exact():
    need_gpu()
    g = np.random.Generator(np.random.PCG64(31))
    h = torch.randn((3000, 4096), device="cuda").to(torch.bfloat16)
    mask = g.random(3000) < 0.5
    r = P.batch_compact(h, torch.from_numpy(mask).cuda())
    e, c = O.compact_indices(mask)
    assert torch.equal(r.exiting, h[torch.from_numpy(e).cuda()])
    assert torch.equal(r.continuing, h[torch.from_numpy(c).cuda()])


def test_projection_golden(golden_projection):
    need_gpu()
    g = golden_projection
    out = np.full((20, 64), -1.0, np.float32)
    P.exit_projection(g["rows"], g["gain"], O.DEFAULT_EPS, g["positions"], out)
    np.testing.assert_allclose(out, g["out"], rtol=2e-6, atol=1e-6)
    out2 = np.full((20, 64), -1.0, np.float32)
    P.exit_projection(g["rows"], None, O.DEFAULT_EPS, g["positions"], out2)
    np.testing.assert_allclose(out2, g["out_nogain"], rtol=2e-6, atol=1e-6)
    # untouched rows preserved exactly
    untouched = np.setdiff1d(np.arange(20), g["positions"])
    assert np.all(out[untouched] == -1.0)


def test_scatter_roundtrip_and_validation(rng):
    need_gpu()
    h = rng.standard_normal((30, 8), dtype=np.float32)
    mask = rng.integers(0, 2, size=30).astype(bool)
    res = P.batch_compact(h, mask)
    out = np.zeros_like(h)
    P.exit_scatter(res.exiting, res.exiting_indices, out)
    P.exit_scatter(res.continuing, res.continuing_indices, out)
    np.testing.assert_array_equal(out, h)
    out = np.zeros((5, 2), np.float32)
    with pytest.raises(ValueError, match="strictly increasing"):
        P.exit_scatter(np.ones((2, 2), np.float32), [3, 1], out)
    with pytest.raises(ValueError, match="strictly increasing"):
        P.exit_scatter(np.ones((2, 2), np.float32), [2, 2], out)
    with pytest.raises(ValueError, match="range"):
        P.exit_scatter(np.ones((2, 2), np.float32), [1, 3], np.zeros((3, 2), np.float32))
    with pytest.raises(ValueError, match="width"):
        P.exit_scatter(np.ones((1, 2), np.float32), [0], np.zeros((3, 4), np.float32))
    keep = np.full((3, 2), 7.0, np.float32)
    P.exit_scatter(np.zeros((0, 2), np.float32), np.zeros(0, np.int64), keep)
    assert np.all(keep == 7.0)


def test_projection_bf16_rows_device():
    need_gpu()
    g = np.random.Generator(np.random.PCG64(41))
    rows = O.round_to(g.standard_normal((257, 4096), dtype=np.float32) * 3, "bf16")
    gain = g.standard_normal(4096, dtype=np.float32)
    pos = np.sort(g.choice(1000, 257, replace=False)).astype(np.int64)
    out = torch.zeros((1000, 4096), dtype=torch.float32, device="cuda")
    P.exit_projection(torch.from_numpy(rows).cuda().to(torch.bfloat16),
                      torch.from_numpy(gain).cuda(), 1e-6, torch.from_numpy(pos).cuda(), out)
    want = np.zeros((1000, 4096), np.float32)
    O.exit_projection(rows, gain, 1e-6, pos, want)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("d", [8, 9, 130, 768, 772, 1000, 4096, 5003, 16384])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_staged_projection_bit_identical(d, dtype, monkeypatch):
    """The staged rmsnorm (row in shared memory, numpy's pairwise tree laid
    out by the host and summed four leaves at a time) == the one-pass
    global-read kernel == the numpy oracle, bit for bit; exit_projection and
    select_project's f32 and bf16-pair stagings."""
    need_gpu()
    import torch
    g = np.random.Generator(np.random.PCG64(d))
    n = 300
    rows = torch.from_numpy(g.standard_normal((n, d), dtype=np.float32) * 3).cuda()
    if dtype == "bf16":
        rows = rows.to(torch.bfloat16)
    gain = (g.standard_normal(d) * 0.5 + 1).astype(np.float32)
    pos = torch.arange(0, 2 * n, 2, dtype=torch.int64, device="cuda")
    outs, st = {}, {}
    lib = N.load()
    ptrs = N.ptr_array([rows.data_ptr()])
    gd = torch.from_numpy(gain).cuda()
    code = N.F32 if dtype == "f32" else N.BF16
    for staged in ("1", "0"):
        monkeypatch.setenv("TIDE_PROJECT_STAGED", staged)
        out = torch.zeros((2 * n, d), device="cuda")
        P.exit_projection(rows, gain, 1e-6, pos, out)
        outs[staged] = out
        f32 = torch.empty((n, d), device="cuda")
        hi = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
        lo = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
        s = D.stream_handle()
        N.check(lib.tide_select_project(ptrs, 1, d, code, None, n, d, gd.data_ptr(), 1e-6,
                                        f32.data_ptr(), d, s), "select_project")
        N.check(lib.tide_select_project_split(ptrs, 1, d, code, None, n, d, gd.data_ptr(), 1e-6,
                                              hi.data_ptr(), lo.data_ptr(), d, s), "split")
        torch.cuda.synchronize()
        st[staged] = (f32, hi, lo)
    assert torch.equal(outs["1"], outs["0"])
    for a, b in zip(st["1"], st["0"]):
        assert torch.equal(a, b)
    want = np.zeros((2 * n, d), np.float32)
    O.exit_projection(rows.float().cpu().numpy(), gain, 1e-6, pos.cpu().numpy(), want)
    np.testing.assert_array_equal(outs["1"].cpu().numpy(), want)


@pytest.mark.parametrize("shape,dtype", [((9000, 4099), np.float32), (((33 << 20) // 8 + 5,), np.int64),
                                         ((70000, 512), np.float32), ((10, 7), np.float32)])
def test_staged_upload_equals_pageable_copy(shape, dtype):
    """Host arrays >= 32 MB reach the device through the two pinned staging
    buffers (_device.upload, chunks of 64 MB, host copy of one chunk under
    the DMA of the previous): byte-identical to torch's pageable copy, for
    sizes that are not a multiple of the chunk; two uploads back to back
    (the second reuses the buffers while the first's DMAs may be in flight),
    and the staged download (_device.to_host) of large results."""
    need_gpu()
    Dv = D
    g = np.random.Generator(np.random.PCG64(sum(shape)))
    a = (g.standard_normal(shape) * 1000).astype(dtype)
    b = (g.standard_normal(shape) * 1000).astype(dtype)
    ta = Dv.upload(a)
    tb = Dv.upload(b)
    torch.cuda.synchronize()
    assert torch.equal(ta.cpu(), torch.from_numpy(a))
    assert torch.equal(tb.cpu(), torch.from_numpy(b))
    # and back: to_host stages large results through the same pair
    tb.mul_(3)  # produced on the stream right before the download
    back = Dv.to_host(tb)
    assert back.dtype == b.dtype and back.shape == b.shape
    assert np.array_equal(back, (torch.from_numpy(b) * 3).numpy())
    mask = Dv.to_host(ta.reshape(-1) > 0)
    assert np.array_equal(mask, a.reshape(-1) > 0)


def test_dropin_host_arrays_through_staging_match_oracle():
    """The reference-facing calls with host arrays large enough for the
    staged H2D / D2H (>= 32 MB): fused_layernorm_route's scores equal the
    device-input call's bitwise (decisions inside the f32 band of the oracle),
    and batch_compact's host row copies / indices equal the oracle's
    batch_compact exactly."""
    need_gpu()
    g = np.random.Generator(np.random.PCG64(123))
    n, d = 9000, 1024  # 36.9 MB of f32 rows
    h = g.standard_normal((n, d), dtype=np.float32)
    orouter = O.make_router(d, 128, 3, g)
    router = P.Router(layer=3, w_down=orouter.w_down, w_up=orouter.w_up)
    s_host = P.fused_layernorm_route(h, router)
    assert isinstance(s_host, np.ndarray) and s_host.dtype == np.float32
    s_dev = P.fused_layernorm_route(torch.from_numpy(h).cuda(), router).cpu().numpy()
    assert np.array_equal(s_host, s_dev)
    _, t_ref, m_ref = O.route_logits(h[:2048], orouter)
    assert O.decision_band_ok(s_host[:2048] > np.float32(0.5), t_ref, m_ref, 0.5, 1e-5).all()
    mask = s_host > np.float32(0.5)
    got = P.batch_compact(h, mask)
    want = O.batch_compact(h, mask)
    for k in ("continuing", "exiting", "continuing_indices", "exiting_indices"):
        a, b = getattr(got, k), getattr(want, k)
        assert isinstance(a, np.ndarray), k
        assert np.array_equal(a, b), k
