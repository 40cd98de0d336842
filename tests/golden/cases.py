"""Seeded input recipes shared by the golden generator and the tests.

Pure numpy; no dependency on the reference.  Every recipe is a function of
its spec (PCG64 seeds), so the inputs are regenerated bit-identically on the
GPU box and checked against the SHA-1 stored in the golden file.
"""

from __future__ import annotations

import ast
import hashlib

import numpy as np


def digest(*arrays) -> str:
    h = hashlib.sha1()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def stored_digest(npz, key) -> str:
    return bytes(npz[key]).decode()


def posthoc_cases(npz):
    """Decode the case table written by make_golden.gen_posthoc."""
    return [ast.literal_eval(c) for c in npz["cases"]]


def bank_from_golden(npz, bname):
    """-> (checkpoints tuple, eps, {k: (w_down, w_up)})"""
    ckpts = tuple(int(k) for k in npz[f"{bname}__ckpts"])
    eps = float(npz[f"{bname}__eps"][0])
    return ckpts, eps, {k: (npz[f"{bname}__wd_{k}"], npz[f"{bname}__wu_{k}"]) for k in ckpts}


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "f32":
        return x
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        u = x.view(np.uint32).astype(np.uint64)
        rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return rounded.astype(np.uint32).view(np.float32)
    raise ValueError(dtype)


def rigged_router_arrays(d: int, hot: bool, scale: float = 64.0):
    """Restates ee/fixtures/__init__.py:42-53 (rows in +/- pairs)."""
    b = 2 * d
    w_down = np.zeros((b, d), dtype=np.float32)
    for i in range(d):
        w_down[2 * i, i] = scale
        w_down[2 * i + 1, i] = -scale
    w_up = np.full((1, b), 1.0 if hot else -1.0, dtype=np.float32)
    return w_down, w_up


# name -> spec.  kind "acc": acceptance-#2 recipe (test_acceptance.py:72-79);
# kind "unit": test_router_ops.py:45-48 recipe; kind "rigged": fixture routers.
ROUTE_CASES = {
    "unit_64x32": dict(kind="unit", n=200, d=64, b=32, seed=1234, hscale=5.0, dtype="f32"),
    "unit_x100": dict(kind="unit", n=50, d=64, b=32, seed=1235, hscale=100.0, dtype="f32"),
    "acc_64x32": dict(kind="acc", n=2000, d=64, b=32, seed=202, dtype="f32"),
    "acc_256x128": dict(kind="acc", n=1000, d=256, b=128, seed=203, dtype="f32"),
    "acc_4096x128": dict(kind="acc", n=300, d=4096, b=128, seed=204, dtype="f32"),
    "gpt2_768x128": dict(kind="acc", n=2048, d=768, b=128, seed=42, dtype="f32"),
    "bf16_4096x128": dict(kind="acc", n=640, d=4096, b=128, seed=205, dtype="bf16"),
    "bf16_768x128": dict(kind="acc", n=700, d=768, b=128, seed=206, dtype="bf16"),
    "bf16_4096x256": dict(kind="acc", n=300, d=4096, b=256, seed=207, dtype="bf16"),
    "bf16_8192x128": dict(kind="acc", n=200, d=8192, b=128, seed=208, dtype="bf16"),
    "f16_4096x128": dict(kind="acc", n=300, d=4096, b=128, seed=209, dtype="f16"),
    "bf16_200x48": dict(kind="acc", n=333, d=200, b=48, seed=210, dtype="bf16"),
    "f32_12x6": dict(kind="acc", n=77, d=12, b=6, seed=211, dtype="f32"),
    "zero_rows_256": dict(kind="acc", n=100, d=256, b=128, seed=212, dtype="bf16",
                          zero_rows=(0, 5, 99)),
    "rigged_hot_64": dict(kind="rigged", n=64, d=64, hot=True, seed=213, hscale=6e-3,
                          dtype="f32", zero_rows=(3,)),
    "rigged_cold_64": dict(kind="rigged", n=64, d=64, hot=False, seed=214, hscale=6e-3,
                           dtype="f32"),
    "rigged_hot_64_bf16": dict(kind="rigged", n=256, d=64, hot=True, seed=215, hscale=1.0,
                               dtype="bf16", zero_rows=(7,)),
}


def make_route_inputs(spec):
    """-> (h [n,d] f32 (already rounded to spec dtype), w_down [b,d] f32, w_up [1,b] f32)."""
    rng = np.random.Generator(np.random.PCG64(spec["seed"]))
    n, d = spec["n"], spec["d"]
    if spec["kind"] == "unit":
        b = spec["b"]
        w_down = rng.standard_normal((b, d), dtype=np.float32)
        w_up = rng.standard_normal((1, b), dtype=np.float32)
        h = rng.standard_normal((n, d), dtype=np.float32) * np.float32(spec["hscale"])
    elif spec["kind"] == "acc":
        b = spec["b"]
        w_down = (rng.standard_normal((b, d)) * 0.05).astype(np.float32)
        w_up = (rng.standard_normal((1, b)) * 0.05).astype(np.float32)
        h = rng.standard_normal((n, d), dtype=np.float32)
    elif spec["kind"] == "rigged":
        w_down, w_up = rigged_router_arrays(d, spec["hot"])
        h = rng.standard_normal((n, d), dtype=np.float32) * np.float32(spec["hscale"])
    else:
        raise ValueError(spec["kind"])
    h = round_to(h, spec["dtype"])
    for r in spec.get("zero_rows", ()):
        h[r] = 0.0
    return np.ascontiguousarray(h), w_down, w_up


LABEL_CASES = {
    "basic_256": dict(n=512, d=256, ckpts=(3, 7, 11), seed=301, noise=0.15, tau=0.98,
                      dtype="f32"),
    "zero_rows": dict(n=64, d=128, ckpts=(3, 7), seed=302, noise=0.1, tau=0.5, dtype="f32",
                      zero_ckpt_rows=((3, 1), (7, 4)), zero_final_rows=(9,)),
    "bf16_4096": dict(n=256, d=4096, ckpts=(3, 7, 11, 15, 19, 23, 27, 31), seed=303,
                      noise=0.14, tau=0.98, dtype="bf16"),
    "bf16_odd": dict(n=129, d=200, ckpts=(3, 7, 11, 15, 19, 23, 27, 31, 35), seed=304,
                     noise=0.3, tau=0.9, dtype="bf16"),
    "straddle": dict(kind="straddle", n=40, d=4, ckpts=(3,), tau=0.98, dtype="f32"),
}


def make_label_inputs(spec):
    """-> (dict layer -> [n,d] f32, final [n,d] f32)."""
    if spec.get("kind") == "straddle":
        # test_calibration.py:155-171: rotations of a fixed vector by known angles
        final = np.zeros((40, 4), dtype=np.float32)
        final[:, 0] = 1.0
        angles = np.linspace(0.0, 0.4, 40)
        ck = np.zeros((40, 4), dtype=np.float32)
        ck[:, 0] = np.cos(angles)
        ck[:, 1] = np.sin(angles)
        return {3: ck}, final
    rng = np.random.Generator(np.random.PCG64(spec["seed"]))
    n, d = spec["n"], spec["d"]
    final = round_to(rng.standard_normal((n, d), dtype=np.float32), spec["dtype"])
    ckpts = {}
    for i, k in enumerate(spec["ckpts"]):
        noise = np.float32(spec["noise"] * (1.0 + 0.25 * i))
        h = final + rng.standard_normal((n, d), dtype=np.float32) * noise
        ckpts[k] = round_to(h, spec["dtype"])
    for k, r in spec.get("zero_ckpt_rows", ()):
        ckpts[k][r] = 0.0
    for r in spec.get("zero_final_rows", ()):
        final[r] = 0.0
    return ckpts, final


def posthoc_states(seed: int, n: int, zero_row=None, num_layers: int = 12, d: int = 64):
    """test_runtime.py:16-19: embedding + one state per layer, N(0,1) f32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    states = [rng.standard_normal((n, d), dtype=np.float32) for _ in range(num_layers + 1)]
    if zero_row is not None:
        states[zero_row[0]][zero_row[1]] = 0.0
    return states
