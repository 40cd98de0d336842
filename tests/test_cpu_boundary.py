"""CPU-only checks: the C-ABI library loads and exports every symbol declared
in include/tide_b200.h with the ctypes signatures the host layer binds; the
host-side API objects validate exactly like the reference; the product path
refuses to run without a GPU (no CPU fallback)."""

import os
import re
import subprocess

import numpy as np
import pytest

import paper_2603_21365_b200 as P
from paper_2603_21365_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tide_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tide_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIBPATH):
        from paper_2603_21365_b200.build import build
        build()
    return N.load()


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 11
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/tide_b200.h but not exported"
        assert name in N.SIGNATURES, f"{name} has no ctypes signature in _native.py"
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIBPATH], capture_output=True,
                         text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_metadata_without_gpu(lib):
    assert lib.tide_version().decode().startswith("tide_b200")
    assert lib.tide_workspace_bytes() == N.WORKSPACE_BYTES
    assert lib.tide_route_uses_tensor_cores(N.BF16, 4096, 128) == 1
    assert lib.tide_route_uses_tensor_cores(N.F32, 4096, 128) == 1  # 3xTF32 (large n)
    assert lib.tide_route_uses_tensor_cores(N.F32, 16384, 128) == 0
    # 3xTF32 only where its measured error stays inside 1e-5 (route_tf32.cu
    # tf32_max_d): narrower bottlenecks average fewer units
    assert lib.tide_route_uses_tensor_cores(N.F32, 8192, 128) == 1
    assert lib.tide_route_uses_tensor_cores(N.F32, 8192, 96) == 0
    assert lib.tide_route_uses_tensor_cores(N.F32, 4096, 64) == 1
    assert lib.tide_route_uses_tensor_cores(N.F32, 4096, 32) == 0
    assert lib.tide_route_uses_tensor_cores(N.F32, 2048, 32) == 1
    assert lib.tide_route_uses_tensor_cores(N.F32, 2048, 16) == 0
    assert lib.tide_route_uses_tensor_cores(N.BF16, 4096, 512) == 0


def test_argument_errors_are_reported_not_computed(lib):
    # shape errors are caught before any device work
    rc = lib.tide_route(None, 0, 10, None, 10, 0, N.BF16, None, None, None, 0, 1e-6, 0.5, 0,
                        None, None, None, None, None, 0, None, None, None, None)
    assert rc == -1
    assert "bad shape" in lib.tide_last_error().decode()
    rc = lib.tide_cos_label(N.ptr_array([0]), 0, None, 0, N.BF16, 1, 1, 0.5, None, None, None,
                            None, None, None)
    assert rc == -1
    # chain tail: bad shape, missing device buffers, unsupported dtype, unordered layers
    one = N.ptr_array([16])
    rc = lib.tide_route_tail(one, 1, 64, 10, 0, N.BF16, 16, 16, 10, 10, one, one, 128,
                             N.i64_array([3]), 1e-6, 0.5, 16, 16, 16, 0, 16, None)
    assert rc == -1 and "bad shape" in lib.tide_last_error().decode()
    rc = lib.tide_route_tail(one, 1, 64, 10, 64, N.BF16, None, 16, 10, 10, one, one, 128,
                             N.i64_array([3]), 1e-6, 0.5, 16, 16, 16, 0, 16, None)
    assert rc == -1 and "null device buffer" in lib.tide_last_error().decode()
    rc = lib.tide_route_tail(one, 1, 64, 10, 64, 7, 16, 16, 10, 10, one, one, 128,
                             N.i64_array([3]), 1e-6, 0.5, 16, 16, 16, 0, 16, None)
    assert rc == -1 and "bad dtype" in lib.tide_last_error().decode()
    two = N.ptr_array([16, 32])
    rc = lib.tide_route_tail(two, 2, 64, 10, 64, N.BF16, 16, 16, 10, 10, two, two, 128,
                             N.i64_array([7, 3]), 1e-6, 0.5, 16, 16, 16, 0, 16, None)
    assert rc == -1 and "unordered layers" in lib.tide_last_error().decode()


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    router = P.Router(layer=3, w_down=np.zeros((4, 8), np.float32),
                      w_up=np.zeros((1, 4), np.float32))
    with pytest.raises(N.NativeUnavailable):
        P.fused_layernorm_route(np.zeros((2, 8), np.float32), router)
    with pytest.raises(N.NativeUnavailable):
        P.batch_compact(np.zeros((2, 8), np.float32), np.zeros(2, bool))


def test_router_validation_matches_reference():
    with pytest.raises(ValueError, match="w_up"):
        P.Router(layer=0, w_down=np.zeros((4, 8), np.float32), w_up=np.zeros((1, 5), np.float32))
    with pytest.raises(ValueError, match="w_down"):
        P.Router(layer=0, w_down=np.zeros(8, np.float32), w_up=np.zeros((1, 8), np.float32))
    r = P.Router(layer=0, w_down=np.zeros((128, 4096), np.float32),
                 w_up=np.zeros((1, 128), np.float32))
    assert r.param_count == 524416 and r.bottleneck == 128 and r.hidden_dim == 4096


@pytest.mark.parametrize("kwargs", [
    {"exit_threshold": 0.0}, {"exit_threshold": 1.2}, {"exit_threshold": -0.5},
    {"k_min": -1}, {"mode": "eager"}, {"max_new_tokens": 0}, {"temperature": -0.1},
])
def test_runtime_config_validation(kwargs):
    with pytest.raises(ValueError):
        P.RuntimeConfig(**kwargs)


def test_runtime_config_defaults():
    cfg = P.RuntimeConfig()
    assert cfg.exit_threshold == 1.0 and cfg.mode == P.PER_TOKEN


def test_checkpoint_layers_formula():
    assert P.checkpoint_layers(32, 4) == (3, 7, 11, 15, 19, 23, 27, 31)
    rng = np.random.Generator(np.random.PCG64(505))
    for _ in range(10):
        L = int(rng.integers(2, 65))
        c = int(rng.integers(1, 17))
        want = tuple(i * c - 1 for i in range(1, L + 1) if i * c - 1 < L)
        assert P.checkpoint_layers(L, c) == want
    with pytest.raises(ValueError):
        P.checkpoint_layers(1, 4)


def test_router_bank_validation():
    wd = np.zeros((8, 16), np.float32)
    wu = np.zeros((1, 8), np.float32)
    bank = P.make_bank({3: (wd, wu), 7: (wd, wu), 11: (wd, wu)}, num_layers=12)
    assert bank.checkpoints == (3, 7, 11) and bank.router_param_count == 16 * 8 + 8
    with pytest.raises(ValueError, match="pattern"):
        P.make_bank({3: (wd, wu), 6: (wd, wu)}, num_layers=12)
    with pytest.raises(ValueError, match="violates"):
        P.RouterBank(hidden_dim=16, bottleneck=4, interval=4, tau=0.98, eps=1e-6, num_layers=12,
                     model_digest=0, routers={k: P.Router(k, wd, wu) for k in (3, 7, 11)},
                     stats={})


def test_phase_stats_histogram():
    st = P.PhaseStats.from_exit_layers([3, -1, 3, 7, -1])
    assert st.tokens_total == 5 and st.exit_rate == pytest.approx(0.6)
    assert st.histogram == {3: 2, "final": 2, 7: 1}
    d = st.to_dict()
    assert list(d["histogram"]) == ["3", "7", "final"]
    assert d["exit_layers"] == [3, None, 3, 7, None]


def test_calibration_config_validation():
    assert P.CalibrationConfig().resolve_bottleneck(4096) == 128
    assert P.CalibrationConfig().resolve_bottleneck(64) == 32
    with pytest.raises(ValueError):
        P.CalibrationConfig(convergence_threshold=1.0)
