"""Shared helpers for the GPU parity tests (oracle = oracle/tide_oracle.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import tide_oracle as O

# north_star tolerances: logits within 1e-5 relative (fp32) / 2e-2 (bf16, fp16),
# relative to the conditioning magnitude m = sum_j |w_up_j a_j|
RTOL = {"f32": 1e-5, "bf16": 2e-2, "f16": 2e-2}
TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def have_gpu() -> bool:
    return torch.cuda.is_available()


def need_gpu():
    if not have_gpu():
        pytest.skip("needs a CUDA device")


def to_dev(h_f32: np.ndarray, dtype: str) -> torch.Tensor:
    """The oracle sees `h_f32` (already rounded to dtype); the GPU gets the same values."""
    t = torch.from_numpy(np.ascontiguousarray(h_f32)).cuda().to(TORCH_DT[dtype])
    back = t.float().cpu().numpy()
    assert np.array_equal(back, h_f32), "rounding recipe and torch disagree"
    return t


def check_logits(t_gpu, t_ref, m_ref, dtype, what=""):
    ok = O.logits_close(t_gpu, t_ref, m_ref, RTOL[dtype])
    if not ok.all():
        i = int(np.argmin(ok))
        rel = np.abs(np.asarray(t_gpu, np.float64) - t_ref) / np.maximum(np.abs(t_ref), m_ref)
        raise AssertionError(f"{what}: {int((~ok).sum())} logits outside band; first row {i}: "
                             f"gpu {t_gpu[i]} ref {t_ref[i]} m {m_ref[i]} max rel {rel.max():.3e}")


def check_decisions(mask_gpu, t_ref, m_ref, theta, dtype, what=""):
    ok = O.decision_band_ok(mask_gpu, t_ref, m_ref, theta, RTOL[dtype])
    assert ok.all(), f"{what}: {int((~ok).sum())} decisions differ outside the band"


def excused_rows(states, routers, theta, dtype, k_min=0):
    """Rows whose exit could legitimately differ: some checkpoint >= k_min has
    an oracle logit inside the band around logit(theta)."""
    n = states[0].shape[0]
    exc = np.zeros(n, bool)
    if float(np.float32(theta)) >= 1.0:
        return exc
    lt = O.logit_of(theta)
    for k, r in routers.items():
        if k < k_min:
            continue
        _, t, m = O.route_logits(states[k + 1], r)
        exc |= np.abs(t.astype(np.float64) - lt) <= RTOL[dtype] * np.maximum(np.abs(t), m)
    return exc
