"""Routing ops on B200 — same names, arguments and errors as
ee/router_ops.py (earlyexit 0.1.0), computed by libtide_b200 kernels.

Host (numpy / list) inputs get host (numpy) results, so the reference's own
tests read unchanged; CUDA tensors stay on the device and results are CUDA
tensors (stream-ordered, no host sync unless the API needs an exact size).
There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .tensor_math import DEFAULT_EPS, as_f32

# ee/router_ops.py:19-21.  Both strategies run the same ballot/prefix kernel;
# they are kept as names because the reference API accepts them.
SMALL_BATCH_CUTOVER = 32
STRATEGIES = ("auto", "small", "prefix")


@dataclass
class Router:
    """Two-layer bottleneck MLP scoring one checkpoint layer (ee/router_ops.py:24-50).

    Weights are kept as f32 host arrays (the reference's format); device
    copies — bf16/f16 [b, d] for the tensor-core kernel, f32 for the CUDA-core
    kernel — are created once per (device, dtype) and cached.
    """

    layer: int
    w_down: np.ndarray  # [b, d]
    w_up: np.ndarray  # [1, b]

    def __post_init__(self):
        self.w_down = as_f32(self.w_down)
        self.w_up = as_f32(self.w_up)
        if self.w_down.ndim != 2:
            raise ValueError(f"w_down must be [b, d], got {self.w_down.shape}")
        if self.w_up.shape != (1, self.w_down.shape[0]):
            raise ValueError(f"w_up must be [1, {self.w_down.shape[0]}], got {self.w_up.shape}")

    @property
    def bottleneck(self) -> int:
        return self.w_down.shape[0]

    @property
    def hidden_dim(self) -> int:
        return self.w_down.shape[1]

    @property
    def param_count(self) -> int:
        return self.w_down.size + self.w_up.size


# device copies of router weights: bounded, identity-checked, weak on the host side
_weight_cache = D.register_cache(D.IdentityCache(256))


def device_weights(router, dtype_code: int, device) -> tuple:
    """(w_down [b, d] in the kernel dtype, w_up [b] f32) on `device`, cached.

    Accepts this package's Router or the reference's (duck-typed).  A cache
    hit needs the same router object holding the same w_down / w_up arrays;
    in-place edits need `invalidate_device_caches()`."""
    dev = torch.device(device)
    wd_host, wu_host = router.w_down, router.w_up
    key = (id(router), dev.index, dtype_code)
    owners = (router, wd_host, wu_host)
    hit = _weight_cache.get(key, owners)
    if hit is not None:
        return hit
    wd32 = torch.from_numpy(np.ascontiguousarray(wd_host, dtype=np.float32)).to(dev)
    if dtype_code == N.BF16:
        wd = wd32.to(torch.bfloat16)
    elif dtype_code == N.F16:
        wd = wd32.to(torch.float16)
    else:
        wd = wd32
    wu = torch.from_numpy(np.ascontiguousarray(wu_host, dtype=np.float32).reshape(-1)).to(dev)
    return _weight_cache.put(key, owners, (wd.contiguous(), wu.contiguous()))


def install_cached(router, dtype_code: int, device, wd: torch.Tensor, wu: torch.Tensor) -> None:
    """Seed the device weight cache with copies made elsewhere (bank_io)."""
    dev = torch.device(device)
    _weight_cache.put((id(router), dev.index, dtype_code), (router, router.w_down, router.w_up),
                      (wd.contiguous(), wu.reshape(-1).contiguous()))


def _rows_for(h, router):
    """Validate like ee/router_ops.py:53-57; -> (device rows, ld, dtype code, host?)."""
    host = D.is_host(h)
    D.require_cuda()
    if host:
        arr = as_f32(h)
        if arr.ndim != 2 or arr.shape[1] != router.hidden_dim:
            raise ValueError(f"expected [batch, {router.hidden_dim}] rows, got {arr.shape}")
        t = D.upload(arr)
    else:
        t = h
        if t.dim() != 2 or t.shape[1] != router.hidden_dim:
            raise ValueError(f"expected [batch, {router.hidden_dim}] rows, got {tuple(t.shape)}")
        if t.dtype not in (torch.float32, torch.float16, torch.bfloat16):
            t = t.float()
    t, ld = D.rows_view(t)
    return t, ld, D.dtype_code(t), host


def route(h, router, eps: float = DEFAULT_EPS, theta: float = 1.0, *, want_scores=True,
          want_logits=False, want_mask=False, want_indices=False, layer=None):
    """One fused launch: scores / logits / mask / stable partition indices.

    Returns a dict of CUDA tensors (indices sliced to exact size: one host
    sync, only when want_indices)."""
    t, ld, code, _ = _rows_for(h, router)
    n, d = t.shape
    dev = t.device
    wd, wu = device_weights(router, code, dev)
    out = {}
    f32 = dict(dtype=torch.float32, device=dev)
    scores = torch.empty(n, **f32) if want_scores else None
    logits = torch.empty(n, **f32) if want_logits else None
    mask = torch.empty(n, dtype=torch.uint8, device=dev) if (want_mask or want_indices) else None
    exit_idx = cont_idx = counts = None
    if want_indices:
        exit_idx = torch.empty(n, dtype=torch.int64, device=dev)
        cont_idx = torch.empty(n, dtype=torch.int64, device=dev)
        counts = torch.empty(2, dtype=torch.int64, device=dev)
    lib = N.load()
    rc = lib.tide_route(t.data_ptr() if n else 0, ld, n, None, n, d, code, None, wd.data_ptr(),
                        wu.data_ptr(), router.bottleneck, float(np.float32(eps)),
                        float(np.float32(theta)), int(layer if layer is not None else router.layer),
                        D.ptr(scores), D.ptr(logits), D.ptr(mask), D.ptr(exit_idx),
                        D.ptr(cont_idx), 0, None, D.ptr(counts), D.workspace(dev).data_ptr(),
                        D.stream_handle(dev))
    N.check(rc, "tide_route")
    if want_scores:
        out["scores"] = scores
    if want_logits:
        out["logits"] = logits
    if want_mask or want_indices:
        out["mask"] = mask.bool()
    if want_indices:
        n_exit = int(counts[0].item())
        out["exiting_indices"] = exit_idx[:n_exit]
        out["continuing_indices"] = cont_idx[: n - n_exit]
    return out


def fused_layernorm_route(h, router, eps: float = DEFAULT_EPS):
    """ee/router_ops.py:68-87: per-row sigmoid(w_up . SiLU((W_down . x) * rsqrt(mean x^2 + eps)))."""
    host = D.is_host(h)
    scores = route(h, router, eps)["scores"]
    return D.to_host(scores) if host else scores


def route_logits(h, router, eps: float = DEFAULT_EPS):
    """Pre-sigmoid logits t of the fused kernel (not in the reference API;
    used by the parity tests' tolerance band)."""
    host = D.is_host(h)
    r = route(h, router, eps, want_scores=True, want_logits=True)
    if host:
        return D.to_host(r["scores"]), D.to_host(r["logits"])
    return r["scores"], r["logits"]


class _NoTF32:
    def __enter__(self):
        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False

    def __exit__(self, *a):
        torch.backends.cuda.matmul.allow_tf32 = self.prev


def route_scores(h, router, eps: float = DEFAULT_EPS):
    """Composed pipeline of ee/router_ops.py:60-65 (rmsnorm -> down -> SiLU ->
    up -> sigmoid) as separate f32 device ops — the equivalence partner of the
    fused kernel, exactly as in the reference."""
    host = D.is_host(h)
    t, _, _, _ = _rows_for(h, router)
    x = t.float()
    z = x / torch.sqrt(torch.mean(x * x, dim=-1, keepdim=True) + np.float32(eps))
    wd, wu = device_weights(router, N.F32, x.device)
    with _NoTF32():
        u = z @ wd.t()
        u = u * torch.sigmoid(u)
        s = torch.sigmoid(u @ wu)
    return D.to_host(s) if host else s


@dataclass
class CompactionResult:
    """ee/router_ops.py:90-97."""

    continuing: object  # [n_cont, d]
    exiting: object  # [n_exit, d]
    continuing_indices: object  # int64, into original batch order
    exiting_indices: object


def _as_mask_dev(exit_mask, batch: int, device):
    if isinstance(exit_mask, torch.Tensor):
        m = exit_mask
        if tuple(m.shape) != (batch,):
            raise ValueError(f"mask length {tuple(m.shape)} does not match batch {batch}")
        return (m != 0).to(device=device, dtype=torch.uint8).contiguous()
    m = np.asarray(exit_mask, dtype=bool)
    if m.shape != (batch,):
        raise ValueError(f"mask length {m.shape} does not match batch {batch}")
    return torch.from_numpy(m.astype(np.uint8)).to(device)


def batch_compact(h, exit_mask, strategy: str = "auto") -> CompactionResult:
    """Stable partition of rows by mask (ee/router_ops.py:137-154), on the
    device: one ordered-look-back kernel for the indices and counts, then the
    same kernel again gathering the rows into exactly-sized outputs."""
    host = D.is_host(h)
    D.require_cuda()
    if host:
        arr = as_f32(h)
        if arr.ndim != 2:
            raise ValueError(f"expected [batch, d] rows, got {arr.shape}")
        t = D.upload(arr)
    else:
        t = h
        if t.dim() != 2:
            raise ValueError(f"expected [batch, d] rows, got {tuple(t.shape)}")
    n, d = t.shape
    mask = _as_mask_dev(exit_mask, n, t.device)
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    t, ld = D.rows_view(t)
    code = D.dtype_code(t)
    dev = t.device
    lib = N.load()
    ws = D.workspace(dev).data_ptr()
    s = D.stream_handle(dev)
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    exit_idx = torch.empty(n, dtype=torch.int64, device=dev)
    cont_idx = torch.empty(n, dtype=torch.int64, device=dev)
    N.check(lib.tide_compact(mask.data_ptr() if n else 0, n, None, None, 0, None, 0, 0, 0,
                             exit_idx.data_ptr(), cont_idx.data_ptr(), None, None,
                             counts.data_ptr(), ws, s), "tide_compact")
    n_exit = int(counts[0].item())
    exiting = torch.empty((n_exit, d), dtype=t.dtype, device=dev)
    continuing = torch.empty((n - n_exit, d), dtype=t.dtype, device=dev)
    if n:
        # indices + counts again (same values) and the rows gathered over those
        # lists by a second, fully parallel kernel
        N.check(lib.tide_compact(mask.data_ptr(), n, None, None, 0, t.data_ptr(), ld, d,
                                 D.elem_bytes(code), exit_idx.data_ptr(), cont_idx.data_ptr(),
                                 exiting.data_ptr() if n_exit else None,
                                 continuing.data_ptr() if n - n_exit else None,
                                 counts.data_ptr(), ws, s), "tide_compact(rows)")
    res = CompactionResult(continuing, exiting, cont_idx[: n - n_exit], exit_idx[:n_exit])
    if host:
        return CompactionResult(*(D.to_host(x) for x in (res.continuing, res.exiting,
                                                         res.continuing_indices,
                                                         res.exiting_indices)))
    return res


def _check_positions(positions, out_rows: int, count: int):
    """ee/router_ops.py:157-167 (same messages)."""
    if isinstance(positions, torch.Tensor):
        p = positions.to(torch.int64)
        if tuple(p.shape) != (count,):
            raise ValueError(f"expected {count} positions, got shape {tuple(p.shape)}")
        if count == 0:
            return p
        if int(p[0]) < 0 or int(p[-1]) >= out_rows:
            raise ValueError(f"positions out of range [0, {out_rows})")
        if count > 1 and bool((p[1:] - p[:-1] <= 0).any()):
            raise ValueError("positions must be strictly increasing")
        return p
    p = np.asarray(positions, dtype=np.int64)
    if p.shape != (count,):
        raise ValueError(f"expected {count} positions, got shape {p.shape}")
    if count == 0:
        return p
    if p[0] < 0 or p[-1] >= out_rows:
        raise ValueError(f"positions out of range [0, {out_rows})")
    if np.any(np.diff(p) <= 0):
        raise ValueError("positions must be strictly increasing")
    return p


def _project(exited, gain, eps, positions, out, normalize: bool, what: str) -> None:
    host_out = D.is_host(out)
    ex_host = D.is_host(exited)
    ex_shape = as_f32(exited).shape if ex_host else tuple(exited.shape)
    out_shape = np.asarray(out).shape if host_out else tuple(out.shape)
    if len(out_shape) != 2 or len(ex_shape) != 2 or ex_shape[1] != out_shape[1]:
        raise ValueError(f"row width mismatch: {ex_shape} into {out_shape}")
    pos = _check_positions(positions, out_shape[0], ex_shape[0])
    if ex_shape[0] == 0 and normalize:
        return
    D.require_cuda()
    rows = D.upload(as_f32(exited)) if ex_host else exited
    rows, ld = D.rows_view(rows)
    dev = rows.device
    if host_out:
        if out.dtype != np.float32:
            raise ValueError("out must be float32")
        dout = torch.from_numpy(np.ascontiguousarray(out)).to(dev)
    else:
        if out.dtype != torch.float32 or out.stride(1) != 1:
            raise ValueError("out must be a float32 row-major tensor")
        dout = out
    dpos = pos.to(dev) if isinstance(pos, torch.Tensor) else torch.from_numpy(pos).to(dev)
    g = None
    if normalize and gain is not None:
        garr = as_f32(gain) if D.is_host(gain) else gain
        gshape = garr.shape if isinstance(garr, np.ndarray) else tuple(garr.shape)
        if tuple(gshape) != (ex_shape[1],):
            raise ValueError(f"gain shape {tuple(gshape)} does not match width {ex_shape[1]}")
        g = D.to_device_f32(garr, dev)
    n_e = ex_shape[0]
    if n_e:
        N.check(N.load().tide_exit_project(rows.data_ptr(), ld, D.dtype_code(rows), None, n_e,
                                           None, ex_shape[1], D.ptr(g), float(np.float32(eps)),
                                           1 if normalize else 0, dpos.data_ptr(),
                                           dout.data_ptr(), dout.stride(0),
                                           D.stream_handle(dev)), what)
    if host_out:
        out[...] = D.to_host(dout)


def exit_scatter(exited, positions, out) -> None:
    """ee/router_ops.py:170-176: copy exited rows back to their positions (in place)."""
    _project(exited, None, DEFAULT_EPS, positions, out, False, "tide_exit_project(scatter)")


def exit_projection(exited, final_norm_gain, eps: float, positions, out) -> None:
    """ee/router_ops.py:179-188: final-norm exited rows into their positions (in place)."""
    _project(exited, final_norm_gain, eps, positions, out, True, "tide_exit_project")
