"""torch.ops.tide.* registrations over the C ABI (the paper's dispatch surface,
PAPER.md:376-392, 413-419: four ops registered via TORCH_LIBRARY).

    import paper_2603_21365_b200.torch_ops  # registers the ops
    scores, logits, mask = torch.ops.tide.fused_layernorm_route(h, w_down, w_up, eps, theta)
    exit_idx, cont_idx, counts = torch.ops.tide.batch_compact(mask)
    torch.ops.tide.exit_scatter(rows, positions, out)
    torch.ops.tide.exit_projection(rows, gain, eps, positions, out)

Device tensors only; the ops launch libtide_b200 kernels on the current
stream (no CPU kernels are registered: calling them on CPU tensors fails).
"""

from __future__ import annotations

import torch

from . import _device as D
from . import _native as N


@torch.library.custom_op("tide::fused_layernorm_route", mutates_args=())
def fused_layernorm_route(h: torch.Tensor, w_down: torch.Tensor, w_up: torch.Tensor,
                          eps: float, theta: float) -> tuple[torch.Tensor, torch.Tensor,
                                                             torch.Tensor]:
    if not h.is_cuda:
        raise RuntimeError("tide::fused_layernorm_route: CUDA tensors only (no CPU fallback)")
    h, ld = D.rows_view(h)
    n, d = h.shape
    b = w_down.shape[0]
    code = D.dtype_code(h)
    wd = w_down.to(h.dtype).contiguous()
    wu = w_up.reshape(-1).float().contiguous()
    scores = torch.empty(n, dtype=torch.float32, device=h.device)
    logits = torch.empty(n, dtype=torch.float32, device=h.device)
    mask = torch.empty(n, dtype=torch.uint8, device=h.device)
    if n:
        N.check(N.load().tide_route(h.data_ptr(), ld, n, None, n, d, code, None, wd.data_ptr(),
                                    wu.data_ptr(), b, eps, theta, 0, scores.data_ptr(),
                                    logits.data_ptr(), mask.data_ptr(), None, None, 0, None,
                                    None, D.workspace(h.device).data_ptr(),
                                    D.stream_handle(h.device)), "tide_route")
    return scores, logits, mask


@fused_layernorm_route.register_fake
def _(h, w_down, w_up, eps, theta):
    n = h.shape[0]
    return (h.new_empty(n, dtype=torch.float32), h.new_empty(n, dtype=torch.float32),
            h.new_empty(n, dtype=torch.uint8))


@torch.library.custom_op("tide::batch_compact", mutates_args=())
def batch_compact(mask: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """-> (exit_idx [n] int64, cont_idx [n] int64, counts [2]); valid prefixes
    exit_idx[:counts[0]], cont_idx[:counts[1]] (no host sync)."""
    if not mask.is_cuda:
        raise RuntimeError("tide::batch_compact: CUDA tensors only (no CPU fallback)")
    m = (mask != 0).to(torch.uint8).contiguous()
    n = m.numel()
    ex = torch.empty(n, dtype=torch.int64, device=m.device)
    co = torch.empty(n, dtype=torch.int64, device=m.device)
    counts = torch.empty(2, dtype=torch.int64, device=m.device)
    N.check(N.load().tide_compact(m.data_ptr() if n else 0, n, None, None, 0, None, 0, 0, 0,
                                  ex.data_ptr(), co.data_ptr(), None, None, counts.data_ptr(),
                                  D.workspace(m.device).data_ptr(), D.stream_handle(m.device)),
            "tide_compact")
    return ex, co, counts


@batch_compact.register_fake
def _(mask):
    n = mask.numel()
    return (mask.new_empty(n, dtype=torch.int64), mask.new_empty(n, dtype=torch.int64),
            mask.new_empty(2, dtype=torch.int64))


def _project(rows, gain, eps, positions, out, normalize):
    rows, ld = D.rows_view(rows)
    n_e, d = rows.shape
    if n_e == 0:
        return
    N.check(N.load().tide_exit_project(rows.data_ptr(), ld, D.dtype_code(rows), None, n_e, None,
                                       d, D.ptr(gain), eps, normalize,
                                       positions.contiguous().data_ptr(), out.data_ptr(),
                                       out.stride(0), D.stream_handle(rows.device)),
            "tide_exit_project")


@torch.library.custom_op("tide::exit_scatter", mutates_args=("out",))
def exit_scatter(rows: torch.Tensor, positions: torch.Tensor, out: torch.Tensor) -> None:
    _project(rows, None, 0.0, positions, out, 0)


@torch.library.custom_op("tide::exit_projection", mutates_args=("out",))
def exit_projection(rows: torch.Tensor, gain: torch.Tensor, eps: float, positions: torch.Tensor,
                    out: torch.Tensor) -> None:
    _project(rows, gain.float().contiguous(), eps, positions, out, 1)
