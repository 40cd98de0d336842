"""Router training on the GPU (ee/calibration.py:222-343).

`train_router(features, labels, layer, config)` is the reference's
signature and contract: the same seeded initialisation (PCG64(seed ^ layer),
N(0,1) * 0.02) and per-epoch permutation stream (drawn on the host from the
same generator, so the minibatch sequence is the reference's), the same
BCE + Adam update, the same errors ("empty", label shape,
TrainingDivergedError naming the layer / epoch / batch offset) and the same
RouterStats.  Features may be a CUDA tensor (e.g. CheckpointCapture output:
collection, labelling and training stay on the device).

Per minibatch: gather z[idx] (z = rmsnorm(features), computed once by the
exit-projection kernel), u = z W^T, d_w_up = g_t a, d_w_down = g_u^T z as f32
library GEMMs (TF32 off), and the two hand-written kernels of
csrc/train.cu for everything elementwise (tide_train_act, tide_adam_step).
The loss of every batch is kept on the device and checked for finiteness once
per epoch, so the loop never synchronises with the host inside an epoch.
Optionally (TIDE_TRAIN_GRAPH=1) one captured CUDA graph of an epoch is
replayed from the second epoch on (the permutation is copied into its static
index buffer, the Adam step index read from device memory).

Results match the reference to f32 rounding of the GEMM summation order (not
bit-exact: BLAS and cuBLAS sum in different orders), see
tests/test_gpu_training.py.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .calibration import FLAG_SINGLE_CLASS, CalibrationConfig, RouterStats
from .router_ops import Router
from .tensor_math import DEFAULT_EPS


class TrainingDivergedError(RuntimeError):
    """Loss went non-finite during router training (ee/calibration.py:40-41)."""


def _rmsnorm_rows(x: torch.Tensor) -> torch.Tensor:
    """z = x / sqrt(mean(x^2) + eps) per row, f32 (tensor_math.rmsnorm, no gain)."""
    n, d = x.shape
    z = torch.empty((n, d), dtype=torch.float32, device=x.device)
    if n:
        pos = torch.arange(n, dtype=torch.int64, device=x.device)
        rows, ld = D.rows_view(x)
        N.check(N.load().tide_exit_project(rows.data_ptr(), ld, D.dtype_code(rows), None, n,
                                           None, d, None, float(np.float32(DEFAULT_EPS)), 1,
                                           pos.data_ptr(), z.data_ptr(), z.stride(0),
                                           D.stream_handle(x.device)), "rmsnorm")
    return z


class _DeviceAdam:
    """_Adam (ee/calibration.py:277-290) over a device f32 tensor.  The bias
    corrections of step t come from a device table (row t - 1) indexed by a
    device step base + a per-batch offset, so one captured epoch replays with
    the right t every epoch."""

    def __init__(self, w: torch.Tensor, config: CalibrationConfig):
        self.w = w
        self.m = torch.zeros_like(w)
        self.v = torch.zeros_like(w)
        f = lambda x: float(np.float32(x))  # noqa: E731
        # Python-scalar arithmetic in f64, rounded to f32 where numpy meets the
        # f32 arrays (NEP 50 weak scalars)
        self.consts = (f(config.adam_beta1), f(1.0 - config.adam_beta1), f(config.adam_beta2),
                       f(1.0 - config.adam_beta2))
        self.lr = f(config.learning_rate)
        self.eps = f(config.adam_eps)

    def step(self, g: torch.Tensor, lib, s, table, step_base, offset: int) -> None:
        N.check(lib.tide_adam_step(self.w.data_ptr(), g.data_ptr(), self.m.data_ptr(),
                                   self.v.data_ptr(), self.w.numel(), *self.consts,
                                   table.data_ptr(), step_base.data_ptr(), offset, 0.0, 0.0,
                                   self.lr, self.eps, s), "tide_adam_step")


def _bias_corrections(config: CalibrationConfig, steps: int) -> np.ndarray:
    """[steps, 2] f32: (1 - beta1^t, 1 - beta2^t) for t = 1..steps, as the
    reference's Python floats round into its f32 arrays."""
    t = np.arange(1, steps + 1, dtype=np.float64)
    out = np.empty((steps, 2), np.float32)
    out[:, 0] = (1.0 - np.power(config.adam_beta1, t)).astype(np.float32)
    out[:, 1] = (1.0 - np.power(config.adam_beta2, t)).astype(np.float32)
    return out


def _as_device_f32(x, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)


def train_router(features, labels, layer: int, config: CalibrationConfig, *, device=None):
    """Train one router on its checkpoint's (row, label) pairs on the GPU.

    Returns (Router, RouterStats) like ee/calibration.py:293-343."""
    n = int(features.shape[0])
    if n == 0:
        raise ValueError("cannot train a router on an empty dataset")
    if tuple(labels.shape) != (n,):
        raise ValueError(f"labels shape {tuple(labels.shape)} does not match {n} rows")
    D.require_cuda()
    if device is None:
        device = features.device if isinstance(features, torch.Tensor) and features.is_cuda \
            else torch.device("cuda", torch.cuda.current_device())
    d = int(features.shape[1])
    b = config.resolve_bottleneck(d)
    rng = np.random.Generator(np.random.PCG64(config.seed ^ layer))
    w_down0 = rng.standard_normal((b, d), dtype=np.float32) * np.float32(0.02)
    w_up0 = rng.standard_normal((1, b), dtype=np.float32) * np.float32(0.02)

    lib = N.load()
    s = D.stream_handle(device)
    x = _as_device_f32(features, device)
    y = _as_device_f32(labels, device)
    z = _rmsnorm_rows(x)
    w_down = torch.from_numpy(w_down0).to(device)
    w_up = torch.from_numpy(w_up0).to(device)
    opt_down, opt_up = _DeviceAdam(w_down, config), _DeviceAdam(w_up, config)
    B = config.batch_size
    nb = (n + B - 1) // B
    # per-batch scratch (sized for a full batch), per-epoch loss record
    u = torch.empty((min(B, n), b), dtype=torch.float32, device=device)
    a = torch.empty_like(u)
    gu = torch.empty_like(u)
    gt = torch.empty(min(B, n), dtype=torch.float32, device=device)
    losses = torch.zeros(nb, dtype=torch.float64, device=device)
    g_down = torch.empty_like(w_down)
    g_up = torch.empty_like(w_up)

    table = torch.from_numpy(_bias_corrections(config, config.epochs * nb)).to(device)
    step_base = torch.zeros(1, dtype=torch.int64, device=device)
    order = torch.empty(n, dtype=torch.int64, device=device)

    def epoch_body():
        st = D.stream_handle(device)  # the capture stream while a graph records
        for bi in range(nb):
            idx = order[bi * B:(bi + 1) * B]
            m = idx.numel()
            zb = z.index_select(0, idx)
            yb = y.index_select(0, idx)
            ub, ab, gub, gtb = u[:m], a[:m], gu[:m], gt[:m]
            torch.matmul(zb, w_down.t(), out=ub)
            N.check(lib.tide_train_act(ub.data_ptr(), m, b, w_up.data_ptr(), yb.data_ptr(),
                                       ab.data_ptr(), gub.data_ptr(), gtb.data_ptr(), None,
                                       ctypes.c_void_p(losses.data_ptr() + 8 * bi), st),
                    "tide_train_act")
            torch.matmul(gtb[None, :], ab, out=g_up)
            torch.matmul(gub.t(), zb, out=g_down)
            opt_down.step(g_down, lib, st, table, step_base, bi)
            opt_up.step(g_up, lib, st, table, step_base, bi)

    # Opt-in (TIDE_TRAIN_GRAPH=1): epoch 0 runs eagerly, later epochs replay
    # one captured epoch.  Measured at 65,536 x 4096, batch 1024: 9.8 ->
    # 8.6 ms per epoch (the batches are GEMM-bound, not launch-bound), against
    # a first capture costing 0.1-1 s, so eager is the default.
    use_graph = config.epochs >= 3 and os.environ.get("TIDE_TRAIN_GRAPH", "0") == "1"
    graph = None
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False  # f32 products, as numpy
    try:
        for epoch in range(config.epochs):
            order.copy_(torch.from_numpy(rng.permutation(n)))
            step_base.fill_(epoch * nb)
            losses.zero_()
            if graph is not None:
                graph.replay()
            else:
                epoch_body()
            ok = torch.isfinite(losses)
            if not bool(ok.all()):
                bad = int((~ok).nonzero()[0, 0])
                raise TrainingDivergedError(
                    f"non-finite loss at layer {layer}, epoch {epoch}, "
                    f"batch offset {bad * B} (lr={config.learning_rate}, "
                    f"batch_size={config.batch_size})")
            if use_graph and graph is None:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    epoch_body()

        # final loss, logits and accuracy over every row (ee/calibration.py:331-343)
        uf = z @ w_down.t()
        t_all = torch.empty(n, dtype=torch.float32, device=device)
        N.check(lib.tide_train_act(uf.data_ptr(), n, b, w_up.data_ptr(), y.data_ptr(), None,
                                   None, None, t_all.data_ptr(), None, s), "tide_train_act")
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    # per-row BCE terms in f32 as the reference forms them, summed in a fixed
    # order (deterministic: test_deterministic compares stats for equality)
    terms = torch.clamp(t_all, min=0.0) - t_all * y + torch.log1p(torch.exp(-t_all.abs()))
    final_loss = float(terms.to(torch.float64).sum().item()) / n
    predictions = (t_all > 0.0).to(torch.float32)
    accuracy = float((predictions == y).to(torch.float64).mean().item())
    positives = int(y.sum().item())
    flags = FLAG_SINGLE_CLASS if positives in (0, n) else 0
    stats = RouterStats(examples=n, positives=positives, final_loss=final_loss,
                        accuracy=accuracy, flags=flags)
    router = Router(layer=layer, w_down=w_down.cpu().numpy(), w_up=w_up.cpu().numpy())
    return router, stats
