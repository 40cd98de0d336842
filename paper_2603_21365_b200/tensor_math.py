"""Numeric primitives of the path (ee/tensor_math.py), device-backed where
they are hot: batched_cosine_similarity runs the labeller kernel."""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _native as N

DEFAULT_EPS = 1e-6  # ee/tensor_math.py:12


def as_f32(x) -> np.ndarray:
    """ee/tensor_math.py:19-21 (host arrays)."""
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(x, dtype=np.float32)


def batched_cosine_similarity(a, b):
    """ee/tensor_math.py:96-113 on the device: (sims [n] f32, zero_mask [n] bool)."""
    host = D.is_host(a) and D.is_host(b)
    D.require_cuda()
    ta = D.upload(as_f32(a)) if D.is_host(a) else a
    tb = D.upload(as_f32(b)) if D.is_host(b) else b
    if tuple(ta.shape) != tuple(tb.shape) or ta.dim() != 2:
        raise ValueError(f"expected matching [n,d] arrays, got {tuple(ta.shape)} and {tuple(tb.shape)}")
    if ta.dtype != tb.dtype:
        ta, tb = ta.float(), tb.float()
    ta, tb = ta.contiguous(), tb.contiguous()
    n, d = ta.shape
    dev = ta.device
    sims = torch.empty(n, dtype=torch.float32, device=dev)
    zero = torch.empty(n, dtype=torch.uint8, device=dev)
    if n:
        N.check(N.load().tide_cos_label(N.ptr_array([ta.data_ptr()]), 1, tb.data_ptr(), d,
                                        D.dtype_code(ta), n, d, 2.0, sims.data_ptr(), None,
                                        None, zero.data_ptr(), None, D.stream_handle(dev)),
                "tide_cos_label")
    zero = zero.bool()
    if host:
        return D.to_host(sims), D.to_host(zero)
    return sims, zero
