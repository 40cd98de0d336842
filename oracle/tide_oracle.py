"""CPU oracle for the TIDE per-token exit-decision hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2603_21365_b200/`) imports this module; only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference`
legs may call it, and only as the checker (or the timed CPU reference arm).

This is a numpy restatement of the reference algorithm (earlyexit 0.1.0,
`/root/reference/pkg/src/earlyexit/`, abbreviated `ee/` below).  The
reference is pure numpy; no third-party arithmetic other than numpy BLAS is
involved.  Every function cites the reference file:line it restates.

Parity is PINNED: `tests/golden/make_golden.py` imports the real reference
(here, in the build container) and writes its outputs on seeded inputs to
`tests/golden/*.npz`; `tests/test_oracle_golden.py` checks this restatement
against those vectors (bit-exact for indices / decisions, tolerance for
floating point, exactly as the reference's own tests pin them).

Additions over the reference (the reference never exposes them):
  * `route_logits` returns the pre-sigmoid logit t and the conditioning
    magnitude m = sum_j |w_up_j * a_j| used by the tolerance band rule.
  * `decision_band_ok` implements the north_star decision rule: GPU exit
    decisions must equal the oracle's except for tokens whose logit lies
    inside rtol*max(|t|, m) of logit(theta).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEFAULT_EPS = 1e-6                    # ee/tensor_math.py:12
SMALL_BATCH_CUTOVER = 32              # ee/router_ops.py:21
NO_EXIT = -1                          # ee/runtime.py:35
PER_TOKEN = "per-token"               # ee/runtime.py:28
BATCH_UNANIMOUS = "batch-unanimous"   # ee/runtime.py:29


def as_f32(x) -> np.ndarray:
    """ee/tensor_math.py:19-21."""
    return np.ascontiguousarray(x, dtype=np.float32)


# ---------------------------------------------------------------------------
# primitives (ee/tensor_math.py)
# ---------------------------------------------------------------------------

def rmsnorm(x, gain=None, eps: float = DEFAULT_EPS) -> np.ndarray:
    """ee/tensor_math.py:35-49: x / sqrt(mean(x^2) + eps) [* gain], f32."""
    x = as_f32(x)
    ms = np.mean(np.square(x), axis=-1, keepdims=True)
    out = x / np.sqrt(ms + np.float32(eps))
    if gain is not None:
        gain = as_f32(gain)
        if gain.shape != (x.shape[-1],):
            raise ValueError(f"gain shape {gain.shape} does not match width {x.shape[-1]}")
        out = out * gain
    return out


def sigmoid(x) -> np.ndarray:
    """ee/tensor_math.py:52-60: two-branch stable logistic in f32."""
    x = as_f32(x)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def silu(x) -> np.ndarray:
    """ee/tensor_math.py:63-66."""
    x = as_f32(x)
    return x * sigmoid(x)


def batched_cosine_similarity(a, b):
    """ee/tensor_math.py:96-113: row cosine, clipped, zero-norm rows -> 0."""
    a = as_f32(a)
    b = as_f32(b)
    if a.shape != b.shape or a.ndim != 2:
        raise ValueError(f"expected matching [n,d] arrays, got {a.shape} and {b.shape}")
    dots = np.einsum("nd,nd->n", a, b)
    na = np.linalg.norm(a, axis=1)
    nb = np.linalg.norm(b, axis=1)
    zero = (na == 0.0) | (nb == 0.0)
    denom = np.where(zero, 1.0, na * nb)
    sims = np.clip(dots / denom, -1.0, 1.0).astype(np.float32)
    sims[zero] = 0.0
    return sims, zero


# ---------------------------------------------------------------------------
# router ops (ee/router_ops.py)
# ---------------------------------------------------------------------------

@dataclass
class OracleRouter:
    """ee/router_ops.py:24-50 (weights f32, w_down [b,d], w_up [1,b])."""
    layer: int
    w_down: np.ndarray
    w_up: np.ndarray

    def __post_init__(self):
        self.w_down = as_f32(self.w_down)
        self.w_up = as_f32(self.w_up)
        if self.w_down.ndim != 2:
            raise ValueError(f"w_down must be [b, d], got {self.w_down.shape}")
        if self.w_up.shape != (1, self.w_down.shape[0]):
            raise ValueError(f"w_up must be [1, {self.w_down.shape[0]}], got {self.w_up.shape}")

    @property
    def bottleneck(self):
        return self.w_down.shape[0]

    @property
    def hidden_dim(self):
        return self.w_down.shape[1]


def _check_width(h, router) -> np.ndarray:
    """ee/router_ops.py:53-57."""
    h = as_f32(h)
    if h.ndim != 2 or h.shape[1] != router.hidden_dim:
        raise ValueError(f"expected [batch, {router.hidden_dim}] rows, got {h.shape}")
    return h


def route_scores(h, router, eps: float = DEFAULT_EPS) -> np.ndarray:
    """Composed pipeline, ee/router_ops.py:60-65."""
    h = _check_width(h, router)
    z = rmsnorm(h, None, eps)
    u = silu(z @ router.w_down.T)
    return sigmoid(u @ router.w_up.T)[:, 0]


def _sigma64(t: float) -> float:
    """ee/router_ops.py:82-86: the final sigmoid is evaluated in f64."""
    if t >= 0.0:
        return 1.0 / (1.0 + math.exp(-t))
    et = math.exp(t)
    return et / (1.0 + et)


def fused_layernorm_route(h, router, eps: float = DEFAULT_EPS) -> np.ndarray:
    """Per-row single pass, ee/router_ops.py:68-87 (loop structure kept)."""
    h = _check_width(h, router)
    n, d = h.shape
    w_down, w_up = router.w_down, router.w_up[0]
    inv_d = np.float32(1.0 / d)
    eps32 = np.float32(eps)
    scores = np.empty(n, dtype=np.float32)
    for i in range(n):
        x = h[i]
        scale = np.float32(1.0) / np.sqrt((x @ x) * inv_d + eps32)
        a = (w_down @ x) * scale
        a *= sigmoid(a)
        t = float(w_up @ a)
        scores[i] = _sigma64(t)
    return scores


def route_logits(h, router, eps: float = DEFAULT_EPS):
    """Same arithmetic as `fused_layernorm_route` (ee/router_ops.py:76-86),
    vectorised over rows, returning (scores f32, logits t f32, m f32) where
    m = sum_j |w_up_j * a_j| is the conditioning magnitude of the logit.

    Vectorising only changes BLAS blocking (gemm instead of gemv), which
    moves the last ulp at most; the golden test pins it to the per-row loop.
    """
    h = _check_width(h, router)
    n, d = h.shape
    inv_d = np.float32(1.0 / d)
    eps32 = np.float32(eps)
    ss = np.einsum("nd,nd->n", h, h).astype(np.float32)
    scale = np.float32(1.0) / np.sqrt(ss * inv_d + eps32)
    a = (h @ router.w_down.T) * scale[:, None]
    a = a * sigmoid(a)
    prod = a * router.w_up[0][None, :]
    t = (a @ router.w_up[0]).astype(np.float32)
    m = np.abs(prod).sum(axis=1).astype(np.float32)
    scores = np.array([_sigma64(float(v)) for v in t], dtype=np.float32)
    return scores, t, m


def logit_of(theta: float) -> float:
    """Inverse of the f64 sigmoid used for the decision threshold."""
    th = float(np.float32(theta))
    if th >= 1.0:
        return math.inf
    return math.log(th / (1.0 - th))


def logits_close(t_gpu, t_ref, m_ref, rtol: float) -> np.ndarray:
    """|t_gpu - t_ref| <= rtol * max(|t_ref|, m)."""
    t_gpu = np.asarray(t_gpu, np.float64)
    t_ref = np.asarray(t_ref, np.float64)
    band = rtol * np.maximum(np.abs(t_ref), np.asarray(m_ref, np.float64))
    return np.abs(t_gpu - t_ref) <= band + 1e-30


def decision_band_ok(mask_gpu, t_ref, m_ref, theta: float, rtol: float) -> np.ndarray:
    """Per token: True when the GPU decision equals `sigma(t_ref) > theta`,
    or the token is excused because |t_ref - logit(theta)| lies inside the
    tolerance band.  theta = 1.0 excuses nobody (nothing may exit)."""
    t_ref = np.asarray(t_ref, np.float64)
    mask_gpu = np.asarray(mask_gpu, bool)
    want = np.array([np.float32(_sigma64(float(v))) > np.float32(theta) for v in t_ref], bool)
    if float(np.float32(theta)) >= 1.0:
        return mask_gpu == want
    band = rtol * np.maximum(np.abs(t_ref), np.asarray(m_ref, np.float64))
    excused = np.abs(t_ref - logit_of(theta)) <= band
    return (mask_gpu == want) | excused


@dataclass
class CompactionResult:
    """ee/router_ops.py:90-97."""
    continuing: np.ndarray
    exiting: np.ndarray
    continuing_indices: np.ndarray
    exiting_indices: np.ndarray


def _as_mask(exit_mask, batch: int) -> np.ndarray:
    """ee/router_ops.py:100-104."""
    mask = np.asarray(exit_mask, dtype=bool)
    if mask.shape != (batch,):
        raise ValueError(f"mask length {mask.shape} does not match batch {batch}")
    return mask


def batch_compact(h, exit_mask, strategy: str = "auto") -> CompactionResult:
    """ee/router_ops.py:107-154.  Both reference strategies produce the same
    stable partition; this restates the prefix-sum path (`:116-134`) and the
    sequential walk (`:107-113`) and dispatches exactly as `:148-154`."""
    h = as_f32(h)
    if h.ndim != 2:
        raise ValueError(f"expected [batch, d] rows, got {h.shape}")
    mask = _as_mask(exit_mask, h.shape[0])
    if strategy == "auto":
        strategy = "small" if h.shape[0] <= SMALL_BATCH_CUTOVER else "prefix"
    if strategy == "small":
        cont = np.asarray([i for i in range(len(mask)) if not mask[i]], dtype=np.int64)
        exi = np.asarray([i for i in range(len(mask)) if mask[i]], dtype=np.int64)
        return CompactionResult(h[cont].copy(), h[exi].copy(), cont, exi)
    if strategy == "prefix":
        n = mask.shape[0]
        ex = mask.astype(np.int64)
        keep = 1 - ex
        exit_dest = np.cumsum(ex) - ex
        keep_dest = np.cumsum(keep) - keep
        n_exit = int(ex.sum())
        cont = np.empty((n - n_exit, h.shape[1]), dtype=h.dtype)
        exi = np.empty((n_exit, h.shape[1]), dtype=h.dtype)
        cont_idx = np.empty(n - n_exit, dtype=np.int64)
        exit_idx = np.empty(n_exit, dtype=np.int64)
        src = np.arange(n, dtype=np.int64)
        cont[keep_dest[~mask]] = h[~mask]
        cont_idx[keep_dest[~mask]] = src[~mask]
        exi[exit_dest[mask]] = h[mask]
        exit_idx[exit_dest[mask]] = src[mask]
        return CompactionResult(cont, exi, cont_idx, exit_idx)
    raise ValueError(f"unknown strategy {strategy!r}")


def compact_indices(mask) -> tuple[np.ndarray, np.ndarray]:
    """Index-only stable partition (the integer part of batch_compact)."""
    mask = np.asarray(mask, bool)
    idx = np.arange(mask.shape[0], dtype=np.int64)
    return idx[mask], idx[~mask]


def _check_positions(positions, out, count: int) -> np.ndarray:
    """ee/router_ops.py:157-167."""
    positions = np.asarray(positions, dtype=np.int64)
    if positions.shape != (count,):
        raise ValueError(f"expected {count} positions, got shape {positions.shape}")
    if count == 0:
        return positions
    if positions[0] < 0 or positions[-1] >= out.shape[0]:
        raise ValueError(f"positions out of range [0, {out.shape[0]})")
    if np.any(np.diff(positions) <= 0):
        raise ValueError("positions must be strictly increasing")
    return positions


def exit_scatter(exited, positions, out) -> None:
    """ee/router_ops.py:170-176."""
    exited = as_f32(exited)
    if out.ndim != 2 or exited.ndim != 2 or exited.shape[1] != out.shape[1]:
        raise ValueError(f"row width mismatch: {exited.shape} into {out.shape}")
    positions = _check_positions(positions, out, exited.shape[0])
    out[positions] = exited


def exit_projection(exited, final_norm_gain, eps, positions, out) -> None:
    """ee/router_ops.py:179-188."""
    exited = as_f32(exited)
    if out.ndim != 2 or exited.ndim != 2 or exited.shape[1] != out.shape[1]:
        raise ValueError(f"row width mismatch: {exited.shape} into {out.shape}")
    positions = _check_positions(positions, out, exited.shape[0])
    if exited.shape[0] == 0:
        return
    out[positions] = rmsnorm(exited, final_norm_gain, eps)


# ---------------------------------------------------------------------------
# checkpoints, labels (ee/calibration.py)
# ---------------------------------------------------------------------------

def checkpoint_layers(num_layers: int, interval: int, include_final: bool = True) -> tuple:
    """ee/calibration.py:86-96."""
    if num_layers < 2 or interval < 1:
        raise ValueError("need num_layers >= 2 and interval >= 1")
    bound = num_layers if include_final else num_layers - 1
    return tuple(k for k in range(interval - 1, bound, interval))


def compute_labels(checkpoint_states: dict, final_states, tau: float):
    """ee/calibration.py:201-219 -> (labels dict f32, sims dict f32, zero_total)."""
    if not 0.0 < tau < 1.0:
        raise ValueError("tau must lie in (0, 1)")
    labels, sims = {}, {}
    zero_total = 0
    for k, h in checkpoint_states.items():
        s, zero = batched_cosine_similarity(h, final_states)
        sims[k] = s
        labels[k] = (s > np.float32(tau)).astype(np.float32)
        zero_total += int(zero.sum())
    return labels, sims, zero_total


# ---------------------------------------------------------------------------
# post-hoc selection (ee/runtime.py:134-181)
# ---------------------------------------------------------------------------

def lm_head_from_hidden(final_norm, lm_head, h) -> np.ndarray:
    """ee/model.py:329-338 with the model reduced to (final_norm, lm_head)."""
    return rmsnorm(as_f32(h), final_norm, DEFAULT_EPS) @ as_f32(lm_head).T


def posthoc_select(final_norm, lm_head, hidden_states, routers: dict, eps: float,
                   theta: float, k_min: int = 0, mode: str = PER_TOKEN,
                   with_logits: bool = True):
    """ee/runtime.py:134-181 (bank checks done by the caller).

    `routers` maps checkpoint layer -> OracleRouter, iterated ascending as
    `RouterBank.checkpoints` (ee/calibration.py:376-378).  Returns
    (logits or None, exit_layers int64)."""
    final_hidden = np.asarray(hidden_states[-1], dtype=np.float32)
    n = final_hidden.shape[0]
    exit_layers = np.full(n, NO_EXIT, dtype=np.int64)
    theta32 = np.float32(theta)
    ckpts = sorted(routers)
    if mode == BATCH_UNANIMOUS:
        for k in ckpts:
            if k < k_min:
                continue
            h_k = np.asarray(hidden_states[k + 1], dtype=np.float32)
            scores = fused_layernorm_route(h_k, routers[k], eps=eps)
            if np.all(scores > theta32):
                exit_layers[:] = k
                logits = lm_head_from_hidden(final_norm, lm_head, h_k) if with_logits else None
                return logits, exit_layers
        logits = lm_head_from_hidden(final_norm, lm_head, final_hidden) if with_logits else None
        return logits, exit_layers
    normed = np.empty_like(final_hidden)
    remaining = np.arange(n, dtype=np.int64)
    for k in ckpts:
        if k < k_min or remaining.size == 0:
            continue
        h_k = np.asarray(hidden_states[k + 1], dtype=np.float32)[remaining]
        scores = fused_layernorm_route(h_k, routers[k], eps=eps)
        mask = scores > theta32
        if not mask.any():
            continue
        parts = batch_compact(h_k, mask)
        exited_at = remaining[parts.exiting_indices]
        exit_projection(parts.exiting, final_norm, DEFAULT_EPS, exited_at, normed)
        exit_layers[exited_at] = k
        remaining = remaining[parts.continuing_indices]
    if remaining.size:
        normed[remaining] = rmsnorm(final_hidden[remaining], final_norm, DEFAULT_EPS)
    logits = normed @ as_f32(lm_head).T if with_logits else None
    return logits, exit_layers


def first_exit_from_scores(scores_by_ckpt: dict, theta: float, k_min: int = 0,
                           mode: str = PER_TOKEN) -> np.ndarray:
    """Exit map implied by per-checkpoint scores: equivalent to the peeling
    loop of ee/runtime.py:164-178 because a row's score at checkpoint k
    depends only on that row (peeling only skips rows that already exited)."""
    theta32 = np.float32(theta)
    ckpts = sorted(scores_by_ckpt)
    n = len(next(iter(scores_by_ckpt.values()))) if ckpts else 0
    out = np.full(n, NO_EXIT, dtype=np.int64)
    if mode == BATCH_UNANIMOUS:
        for k in ckpts:
            if k >= k_min and np.all(np.asarray(scores_by_ckpt[k]) > theta32):
                out[:] = k
                return out
        return out
    for k in ckpts:
        if k < k_min:
            continue
        fire = (np.asarray(scores_by_ckpt[k]) > theta32) & (out == NO_EXIT)
        out[fire] = k
    return out


# ---------------------------------------------------------------------------
# seeded synthetic inputs, shared by tests, smoke and bench
# ---------------------------------------------------------------------------

def make_router(d: int, b: int, layer: int, rng, scale: float = 0.05) -> OracleRouter:
    """Acceptance-#2 recipe (ee tests/test_acceptance.py:72-78): N(0,1)*0.05."""
    return OracleRouter(layer=layer,
                        w_down=(rng.standard_normal((b, d)) * scale).astype(np.float32),
                        w_up=(rng.standard_normal((1, b)) * scale).astype(np.float32))


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round f32 to bf16/f16 and back (the oracle sees the rounded values)."""
    x = as_f32(x)
    if dtype == "f32":
        return x
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        u = x.view(np.uint32).astype(np.uint64)
        # round-to-nearest-even on the top 16 bits
        rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return rounded.astype(np.uint32).view(np.float32)
    raise ValueError(dtype)
