"""Router bank objects and the calibration labeller (ee/calibration.py).

The bank / checkpoint objects keep the reference's fields and validation, so
a reference `earlyexit.RouterBank` and this one are interchangeable inputs to
`posthoc_select`.  `compute_labels` runs the one-pass cosine labeller kernel
over every checkpoint at once.  Router training runs on the GPU in
training.py; hidden-state collection through the
reference's stand-in transformer is out of scope (the CheckpointCapture hook
collects from a real model instead).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .router_ops import Router

BANK_MAGIC = b"TIDE"   # ee/calibration.py:30
BANK_VERSION = 1       # ee/calibration.py:31
FLAG_SINGLE_CLASS = 0x1


def checkpoint_layers(num_layers: int, interval: int, include_final: bool = True) -> tuple:
    """Layers hosting routers, {c-1, 2c-1, ...} below the bound (ee/calibration.py:86-96)."""
    if num_layers < 2 or interval < 1:
        raise ValueError("need num_layers >= 2 and interval >= 1")
    bound = num_layers if include_final else num_layers - 1
    return tuple(k for k in range(interval - 1, bound, interval))


@dataclass(frozen=True)
class CalibrationConfig:
    """Calibration knobs (ee/calibration.py:45-83); validated identically."""

    checkpoint_interval: int = 4
    convergence_threshold: float = 0.98
    bottleneck: Optional[int] = None
    learning_rate: float = 1e-3
    epochs: int = 100
    batch_size: int = 1024
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    seed: int = 0

    def __post_init__(self):
        if self.checkpoint_interval < 1:
            raise ValueError("checkpoint_interval must be >= 1")
        if not 0.0 < self.convergence_threshold < 1.0:
            raise ValueError("convergence_threshold must lie in (0, 1)")
        if self.bottleneck is not None and self.bottleneck < 1:
            raise ValueError("bottleneck must be >= 1")
        if self.learning_rate <= 0 or self.epochs < 1 or self.batch_size < 1:
            raise ValueError("learning_rate, epochs, batch_size must be positive")
        if not (0.0 <= self.adam_beta1 < 1.0 and 0.0 <= self.adam_beta2 < 1.0):
            raise ValueError("adam betas must lie in [0, 1)")
        if self.adam_eps <= 0:
            raise ValueError("adam_eps must be positive")
        if not 0 <= self.seed < 2**64:
            raise ValueError("seed must fit in 64 bits")

    def resolve_bottleneck(self, hidden_dim: int) -> int:
        if self.bottleneck is not None:
            return self.bottleneck
        return min(128, max(1, hidden_dim // 2))


@dataclass
class RouterStats:
    """ee/calibration.py:264-274."""

    examples: int
    positives: int
    final_loss: float
    accuracy: float
    flags: int


@dataclass(eq=False)
class RouterBank:
    """Ascending checkpoint -> Router map with bank metadata (ee/calibration.py:351-382)."""

    hidden_dim: int
    bottleneck: int
    interval: int
    tau: float
    eps: float
    num_layers: int
    model_digest: int
    routers: dict
    stats: dict

    def __post_init__(self):
        layers = self.checkpoints
        expected_with = checkpoint_layers(self.num_layers, self.interval, True)
        expected_without = checkpoint_layers(self.num_layers, self.interval, False)
        if layers not in (expected_with, expected_without):
            raise ValueError(
                f"checkpoint layers {layers} do not follow the interval-{self.interval} "
                f"pattern for {self.num_layers} layers")
        for k, router in self.routers.items():
            if router.w_down.shape != (self.bottleneck, self.hidden_dim):
                raise ValueError(f"router {k} weight shape {router.w_down.shape} "
                                 f"violates bank metadata")

    @property
    def checkpoints(self) -> tuple:
        return tuple(sorted(self.routers))

    @property
    def router_param_count(self) -> int:
        return self.hidden_dim * self.bottleneck + self.bottleneck


def make_bank(routers: dict, num_layers: int, interval: int = 4, eps: float = 1e-6,
              tau: float = 0.98, model_digest: int = 0) -> RouterBank:
    """Convenience constructor from {layer: (w_down, w_up)} or {layer: Router}."""
    rs = {}
    for k, r in routers.items():
        rs[int(k)] = r if hasattr(r, "w_down") else Router(layer=int(k), w_down=r[0], w_up=r[1])
    any_r = next(iter(rs.values()))
    stats = {k: RouterStats(0, 0, 0.0, 1.0, 0) for k in rs}
    return RouterBank(hidden_dim=any_r.hidden_dim, bottleneck=any_r.bottleneck,
                      interval=interval, tau=tau, eps=eps, num_layers=num_layers,
                      model_digest=model_digest, routers=rs, stats=stats)


@dataclass
class CollectedStates:
    """ee/calibration.py:104-109 (arrays may be host numpy or CUDA tensors)."""

    checkpoint_states: dict
    final_states: object
    token_count: int
    corpus_digest: str


@dataclass
class CalibrationDataset:
    """ee/calibration.py:191-198."""

    features: dict
    labels: dict
    similarities: dict
    token_count: int
    corpus_digest: str
    zero_norm_count: int


def label_tensors(checkpoint_states: dict, final_states, tau: float, *, labels_dtype="f32"):
    """The labeller on device tensors, one launch for every checkpoint.

    -> (layers tuple, sims [C, n] f32, labels [C, n] (f32 or u8), zero_counts [C] int64),
    all CUDA tensors, no host sync."""
    if not 0.0 < tau < 1.0:
        raise ValueError("tau must lie in (0, 1)")
    D.require_cuda()
    layers = tuple(checkpoint_states)
    fin = final_states if not D.is_host(final_states) else D.to_device_f32(final_states)
    if fin.dim() != 2:
        raise ValueError(f"expected [n, d] final states, got {tuple(fin.shape)}")
    dev = fin.device
    cks = []
    for k in layers:
        h = checkpoint_states[k]
        h = h if not D.is_host(h) else D.to_device_f32(h, dev)
        if tuple(h.shape) != tuple(fin.shape):
            raise ValueError(f"expected matching [n,d] arrays, got {tuple(h.shape)} and "
                             f"{tuple(fin.shape)}")
        cks.append(h)
    dts = {t.dtype for t in cks} | {fin.dtype}
    if len(dts) != 1:
        fin = fin.float()
        cks = [t.float() for t in cks]
    fin = fin.contiguous()
    cks = [t.contiguous() for t in cks]
    n, d = fin.shape
    C = len(cks)
    sims = torch.empty((C, n), dtype=torch.float32, device=dev)
    lab_f = torch.empty((C, n), dtype=torch.float32, device=dev) if labels_dtype == "f32" else None
    lab_u = torch.empty((C, n), dtype=torch.uint8, device=dev) if labels_dtype == "u8" else None
    zero = torch.empty(C, dtype=torch.int64, device=dev)
    if C:
        N.check(N.load().tide_cos_label(N.ptr_array([t.data_ptr() for t in cks]), C,
                                        fin.data_ptr(), d, D.dtype_code(fin), n, d,
                                        float(np.float32(tau)), sims.data_ptr(), D.ptr(lab_u),
                                        D.ptr(lab_f), None, zero.data_ptr(),
                                        D.stream_handle(dev)), "tide_cos_label")
    return layers, sims, (lab_f if lab_f is not None else lab_u), zero


def compute_labels(states: CollectedStates, tau: float) -> CalibrationDataset:
    """Label each token 1 iff cos(h_k, h_final) > tau, strictly (ee/calibration.py:201-219).

    Zero-norm rows get similarity 0 and label 0 and are counted.  Host inputs
    give host (numpy) labels/similarities; device inputs stay on the device."""
    if not 0.0 < tau < 1.0:
        raise ValueError("tau must lie in (0, 1)")
    host = D.is_host(states.final_states)
    layers, sims, labels, zero = label_tensors(states.checkpoint_states, states.final_states, tau)
    zero_total = int(zero.sum().item()) if len(layers) else 0
    if host:
        sims_h, labels_h = D.to_host(sims), D.to_host(labels)
        sd = {k: sims_h[i] for i, k in enumerate(layers)}
        ld = {k: labels_h[i] for i, k in enumerate(layers)}
    else:
        sd = {k: sims[i] for i, k in enumerate(layers)}
        ld = {k: labels[i] for i, k in enumerate(layers)}
    return CalibrationDataset(features=states.checkpoint_states, labels=ld, similarities=sd,
                              token_count=states.token_count,
                              corpus_digest=states.corpus_digest, zero_norm_count=zero_total)
