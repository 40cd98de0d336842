"""Device plumbing for the host API: tensors in/out, dtype codes, per-stream
workspaces.  PyTorch is used only for device memory and streams."""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _native as N

_TORCH_DT = {torch.float32: N.F32, torch.float16: N.F16, torch.bfloat16: N.BF16}
_ELEM = {N.F32: 4, N.F16: 2, N.BF16: 2}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device visible: the TIDE B200 ops have no CPU fallback")
    N.load()


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _TORCH_DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}; expected float32, float16 or bfloat16")


def elem_bytes(code: int) -> int:
    return _ELEM[code]


def is_host(x) -> bool:
    return not (isinstance(x, torch.Tensor) and x.is_cuda)


def to_device_f32(x, device=None) -> torch.Tensor:
    """Host array-like -> contiguous f32 CUDA tensor (the reference's as_f32)."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if not t.is_cuda:
            t = t.to(device or "cuda")
        if t.dtype not in _TORCH_DT:
            t = t.float()
        return t.contiguous()
    arr = np.ascontiguousarray(x, dtype=np.float32)
    t = torch.from_numpy(arr)
    return t.to(device or "cuda", non_blocking=False)


def rows_view(t: torch.Tensor):
    """-> (tensor, ld) with unit stride along the row; copies only if needed."""
    if t.dim() != 2:
        raise ValueError(f"expected [batch, d] rows, got {tuple(t.shape)}")
    if t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        t = t.contiguous()
    ld = t.stride(0) if t.shape[0] > 1 else t.shape[1]
    return t, max(ld, t.shape[1])


def stream_handle(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_ws_lock = threading.Lock()
_workspaces: dict = {}


def workspace(device=None, stream: int = None) -> torch.Tensor:
    """The look-back workspace of the current stream (allocated + zeroed once).
    `stream` (the raw handle, when the caller already has it) saves a lookup."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    s = stream_handle(dev) if stream is None else stream
    key = (dev.index, s)
    ws = _workspaces.get(key)
    if ws is not None:
        return ws
    with _ws_lock:
        ws = _workspaces.get(key)
        if ws is None:
            ws = torch.empty(N.WORKSPACE_BYTES, dtype=torch.uint8, device=dev)
            N.check(N.load().tide_workspace_init(ws.data_ptr(), s), "tide_workspace_init")
            _workspaces[key] = ws
    return ws


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
