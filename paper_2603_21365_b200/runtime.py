"""Post-hoc exit selection on B200 (ee/runtime.py:28-181).

`posthoc_select` keeps the reference signature and results:
(logits [n, vocab] f32, exit_layers [n] int64, NO_EXIT = -1).  On the device:

  * per-token, n > 16: one fused route+compact launch per checkpoint >= k_min;
    checkpoint k+1 gathers only the rows still remaining (TMA tile::gather4 on
    the previous launch's continuing indices) and reads the remaining count
    from device memory, so the chain never syncs the host;
  * n <= 16 (decode): every checkpoint in ONE launch + in-kernel resolution
    (a row's score at checkpoint k depends only on that row, so the first
    firing checkpoint is exactly what peeling computes);
  * batch-unanimous, n > 16: one launch per checkpoint until all rows fire;
  * then one select_project launch final-norms every row from its exit layer
    (exit_projection + the final-rows rmsnorm of ee/runtime.py:176,180) into
    the bf16-pair operand of the tensor-core LM head (tide_lm_head, 3 MMA
    terms, f32-grade logits).

`model` is anything with .config.num_layers, .config.hidden_dim, .final_norm
and .lm_head — the reference's ReferenceModel, or `OutputHead` below.  `bank`
is this package's RouterBank or the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .router_ops import device_weights
from .tensor_math import DEFAULT_EPS

PER_TOKEN = "per-token"
BATCH_UNANIMOUS = "batch-unanimous"
MODES = (PER_TOKEN, BATCH_UNANIMOUS)
FINAL_KEY = "final"
NO_EXIT = -1


@dataclass(frozen=True)
class RuntimeConfig:
    """ee/runtime.py:38-56 (same validation)."""

    exit_threshold: float = 1.0
    k_min: int = 0
    mode: str = PER_TOKEN
    max_new_tokens: int = 64
    temperature: float = 0.0

    def __post_init__(self):
        if not 0.0 < self.exit_threshold <= 1.0:
            raise ValueError("exit_threshold must lie in (0, 1]")
        if self.k_min < 0:
            raise ValueError("k_min must be >= 0")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.max_new_tokens < 1:
            raise ValueError("max_new_tokens must be >= 1")
        if self.temperature < 0.0:
            raise ValueError("temperature must be >= 0")


@dataclass
class PhaseStats:
    """Exit accounting for one phase (ee/runtime.py:59-92)."""

    tokens_total: int
    exit_layers: list
    histogram: dict
    exit_rate: float

    @classmethod
    def from_exit_layers(cls, exit_layers: Sequence[int]) -> "PhaseStats":
        if isinstance(exit_layers, torch.Tensor):
            exit_layers = exit_layers.detach().cpu().tolist()
        layers = [int(k) for k in exit_layers]
        histogram: dict = {}
        for k in layers:
            key = FINAL_KEY if k == NO_EXIT else k
            histogram[key] = histogram.get(key, 0) + 1
        exited = sum(1 for k in layers if k != NO_EXIT)
        total = len(layers)
        return cls(tokens_total=total, exit_layers=layers, histogram=histogram,
                   exit_rate=(exited / total) if total else 0.0)

    def to_dict(self) -> dict:
        histogram = {str(key): self.histogram[key]
                     for key in sorted(self.histogram,
                                       key=lambda k: (1, 0) if k == FINAL_KEY else (0, k))}
        return {"tokens_total": self.tokens_total, "exit_rate": self.exit_rate,
                "histogram": histogram,
                "exit_layers": [None if k == NO_EXIT else k for k in self.exit_layers]}


@dataclass
class OutputHead:
    """The part of a model posthoc_select touches: depth, width, final norm gain, LM head."""

    num_layers: int
    hidden_dim: int
    final_norm: object  # [d]
    lm_head: object  # [vocab, d]

    @property
    def config(self):
        return self


# LM heads can be GBs: a handful of entries, weak on the host objects
_head_cache = D.register_cache(D.IdentityCache(4))


def _pad8(d: int) -> int:
    return (d + 7) // 8 * 8


def split_bf16(x: torch.Tensor, ld: int):
    """f32 [r, d] -> bf16 pair (hi, lo) [r, ld] (zero-padded columns): hi =
    bf16(x), lo = bf16(x - hi); x - hi is exact in f32, so x = hi + lo to
    ~2^-17 relative (the B operand of tide_lm_head)."""
    r, d = x.shape
    hi = torch.zeros((r, ld), dtype=torch.bfloat16, device=x.device)
    lo = torch.zeros((r, ld), dtype=torch.bfloat16, device=x.device)
    hi[:, :d] = x.to(torch.bfloat16)
    lo[:, :d] = (x - hi[:, :d].float()).to(torch.bfloat16)
    return hi, lo


def _device_head(model, dev):
    """(final-norm gain f32 [d], LM head as the bf16 pair (hi, lo) [vocab, ld])."""
    key = (id(model), dev.index)
    fn, lm = model.final_norm, model.lm_head
    owners = (model, fn, lm)
    hit = _head_cache.get(key, owners)
    if hit is not None:
        return hit
    g = D.to_device_f32(fn, dev).reshape(-1)
    w = D.to_device_f32(lm, dev)
    hi, lo = split_bf16(w, _pad8(w.shape[1]))
    del w
    return _head_cache.put(key, owners, (g, hi, lo))


def lm_head_logits(staged_ptrs, dtype_code, exit_layers, n, d, gain, w_hi, w_lo, dev, s,
                   eps=DEFAULT_EPS):
    """select_project (every row final-normed from its exit layer, written as
    the bf16 pair) + the tensor-core LM head: logits [n, vocab] f32."""
    lib = N.load()
    V = w_hi.shape[0]
    ld = w_hi.shape[1]
    a_hi = torch.empty((n, ld), dtype=torch.bfloat16, device=dev)
    a_lo = torch.empty((n, ld), dtype=torch.bfloat16, device=dev)
    if ld != d:
        a_hi[:, d:].zero_()
        a_lo[:, d:].zero_()
    logits = torch.empty((n, _pad4(V)), dtype=torch.float32, device=dev)
    if n:
        N.check(lib.tide_select_project_split(
            N.ptr_array(staged_ptrs), len(staged_ptrs), d, dtype_code, exit_layers.data_ptr(), n,
            d, gain.data_ptr(), float(np.float32(eps)), a_hi.data_ptr(), a_lo.data_ptr(), ld, s),
            "tide_select_project_split")
        N.check(lib.tide_lm_head(a_hi.data_ptr(), a_lo.data_ptr(), ld, n, d, w_hi.data_ptr(),
                                 w_lo.data_ptr(), ld, V, logits.data_ptr(), logits.shape[1], s),
                "tide_lm_head")
    return logits[:, :V] if logits.shape[1] != V else logits


def _pad4(v: int) -> int:
    return (v + 3) // 4 * 4


def _check_bank(model, hidden_states, bank) -> None:
    """ee/runtime.py:120-131 (same messages)."""
    if len(hidden_states) != bank.num_layers + 1:
        raise ValueError(
            f"got {len(hidden_states)} hidden states, bank expects "
            f"{bank.num_layers + 1} (embedding + one per layer)")
    if hidden_states[0].shape[-1] != bank.hidden_dim:
        raise ValueError(
            f"hidden width {hidden_states[0].shape[-1]} != bank width {bank.hidden_dim}")
    if model.config.num_layers != bank.num_layers:
        raise ValueError(
            f"model has {model.config.num_layers} layers, bank was calibrated for "
            f"{bank.num_layers}")


def _stage_layers(hidden_states, needed: Sequence[int]):
    """Device tensors for the capture indices in `needed`, one common dtype."""
    fast = {}
    dt = None
    for i in needed:
        h = hidden_states[i]
        if (type(h) is not torch.Tensor or not h.is_cuda or h.dim() != 2
                or not h.is_contiguous() or (dt is not None and h.dtype != dt)):
            break
        dt = h.dtype
        fast[i] = h
    else:
        if dt in (torch.float32, torch.float16, torch.bfloat16):
            _check_same_shape(fast, needed)
            return fast, fast[needed[0]].device
    dev = None
    for h in hidden_states:
        if isinstance(h, torch.Tensor) and h.is_cuda:
            dev = h.device
            break
    dev = dev or torch.device("cuda", torch.cuda.current_device())
    out = {}
    for i in needed:
        h = hidden_states[i]
        t = D.to_device_f32(h, dev) if D.is_host(h) else h
        if t.dtype not in (torch.float32, torch.float16, torch.bfloat16):
            t = t.float()
        out[i] = t
    if len({t.dtype for t in out.values()}) > 1:
        out = {i: t.float() for i, t in out.items()}
    for i, t in out.items():
        if t.dim() != 2:
            raise ValueError(f"hidden state {i} must be [n, d], got {tuple(t.shape)}")
        out[i] = t.contiguous()
    _check_same_shape(out, needed)
    return out, dev


def _check_same_shape(staged, needed) -> None:
    """Every kernel reads each capture with the final capture's n, d and ld,
    so a shorter or narrower checkpoint tensor would be read out of bounds;
    the reference fails on it too (ee/runtime.py:166-178 indexes every
    capture with the final batch's row ids: IndexError / ValueError)."""
    ref_i = needed[-1]
    want = tuple(staged[ref_i].shape)
    for i in needed:
        got = tuple(staged[i].shape)
        if got != want:
            raise ValueError(f"hidden state {i} has shape {got}, expected {want} "
                             f"(the shape of hidden state {ref_i})")


_decode_plans = D.register_cache(D.IdentityCache(32))

# limits of the one-launch decode kernel (decode.cu kDMaxC / kDMaxB); other
# shapes take the per-checkpoint chain
MAX_DECODE_CKPTS = 64
MAX_DECODE_B = 256
MAX_TAIL_CKPTS = 32  # route_simt.cu kSimtTailC / route_tcs.cu kMaxTailC


def _decode_plan(bank, ckpts, code, dev):
    """ctypes argument arrays of the decode launch (weight pointers, layers)
    and the device tensors they point into, cached per (bank, checkpoints,
    dtype, device); rebuilt when a router or its weights are replaced.  The
    caller keeps the returned tuple alive as long as it uses the pointers."""
    routers = [bank.routers[k] for k in ckpts]
    key = (id(bank), tuple(ckpts), code, dev.index)
    owners = (bank, *routers, *(r.w_down for r in routers), *(r.w_up for r in routers))
    hit = _decode_plans.get(key, owners)
    if hit is not None:
        return hit
    ws_w = [device_weights(r, code, dev) for r in routers]
    # W of all checkpoints stacked [C, b, d]: the decode kernel then loads its
    # slices with one TMA tensor map (tide_route_decode detects the layout)
    stacked = torch.stack([w for w, _ in ws_w]).contiguous()
    step = stacked[0].numel() * stacked.element_size()
    base = stacked.data_ptr()
    w_arr = N.ptr_array([base + i * step for i in range(len(routers))])
    # bf16 / f16: the routers' W in the decode kernel's shared-memory image,
    # packed once (the kernel fetches its slices with 1-D bulk copies)
    packed = None
    if code != N.F32 and stacked.shape[2] % 8 == 0:
        lib = N.load()
        C, b, d = stacked.shape
        packed = torch.empty(lib.tide_decode_packed_bytes(C, d, b), dtype=torch.uint8, device=dev)
        N.check(lib.tide_decode_pack_weights(w_arr, C, d, b, code, packed.data_ptr(),
                                             D.stream_handle(dev)), "tide_decode_pack_weights")
    arrays = (w_arr, N.ptr_array([u.data_ptr() for _, u in ws_w]), N.i64_array(ckpts),
              packed.data_ptr() if packed is not None else None)
    return _decode_plans.put(key, owners, arrays + ((ws_w, stacked, packed),))


def _decode_ok(n, d, code, b, ckpts, staged) -> bool:
    vec = 4 if code == N.F32 else 8
    return (0 < n <= N.MAX_DECODE_ROWS and 1 <= len(ckpts) <= MAX_DECODE_CKPTS
            and b <= MAX_DECODE_B and d % vec == 0
            and all(staged[k + 1].data_ptr() % 16 == 0 for k in ckpts))


class _ChainGraphs:
    """Replay cache of per-token peeling chains.

    The chain is several launches per call (one per checkpoint, the tail,
    its resolve) whose host issue cost (~130 us at config 2) exceeds their
    device time (~93 us).  The second eager call with the same capture
    buffers (device pointers, shapes, dtype), bank routers and config records
    the chain into a CUDA graph; later calls replay it and return a copy of
    its output.  The key holds the data pointers only, so a replay reads
    whatever the caller's tensors at those addresses hold now — the same
    contract as a captured model step."""

    def __init__(self, size: int = 8):
        from collections import OrderedDict
        self.size = size
        self.entries = OrderedDict()   # key -> [calls, graph, output, keepalive]
        self.streams = {}

    @staticmethod
    def enabled() -> bool:
        import os
        return os.environ.get("TIDE_CHAIN_GRAPHS", "1") != "0"

    @staticmethod
    def knobs() -> tuple:
        """Environment switches that change the recorded launch sequence."""
        import os
        e = os.environ
        return tuple(e.get(k) for k in ("TIDE_CHAIN_TAIL", "TIDE_TAIL_AFTER", "TIDE_TAIL_ROWS",
                                        "TIDE_TAIL_WIDE", "TIDE_SPECULATIVE", "TIDE_WINDOW",
                                        "TIDE_TAIL_KS", "TIDE_SPLIT", "TIDE_PDL",
                                        "TIDE_F32_TAIL_ROWS"))

    def stream(self, dev):
        st = self.streams.get(dev.index)
        if st is None:
            st = self.streams[dev.index] = torch.cuda.Stream(dev)
        return st

    @staticmethod
    def workspace(dev) -> torch.Tensor:
        """A look-back workspace owned by ONE recorded graph.  Graphs recorded
        for different caller streams may replay concurrently; a workspace may
        only be shared by launches that are stream-ordered (common.cuh), so
        every graph gets its own (allocated and zeroed outside the capture)."""
        ws = torch.empty(N.WORKSPACE_BYTES, dtype=torch.uint8, device=dev)
        N.check(N.load().tide_workspace_init(ws.data_ptr(), D.stream_handle(dev)),
                "tide_workspace_init")
        return ws

    def clear(self):
        self.entries.clear()


_chain_graphs = D.register_cache(_ChainGraphs())


def select_exits(hidden_states, bank, config: RuntimeConfig, *, n_rows=None,
                 staged=None, dev=None):
    """Exit map only (int64 CUDA tensor [n]); the hot path of posthoc_select."""
    L = bank.num_layers
    ckpts = [k for k in bank.checkpoints if k >= config.k_min]
    if staged is None:
        staged, dev = _stage_layers(hidden_states, [k + 1 for k in ckpts] + [L])
    final = staged[L]
    n = final.shape[0]
    code = D.dtype_code(final)
    b = _bottleneck(bank, ckpts)
    if ckpts and _decode_ok(n, final.shape[1], code, b, ckpts, staged):
        # decode step: the bound launch of these buffers / routers / config,
        # built once (the argument block of tide_route_decode minus the
        # output pointer), then one ctypes call per step
        s = D.stream_handle(dev)
        routers = [bank.routers[k] for k in ckpts]
        key = (id(bank), tuple(ckpts), float(config.exit_threshold), config.mode,
               config.k_min, final.dtype, tuple(final.shape), s,
               tuple(staged[k + 1].data_ptr() for k in ckpts))
        owners = (bank, *routers, *(r.w_down for r in routers), *(r.w_up for r in routers))
        hit = _decode_calls.get(key, owners)
        if hit is None:
            hit = _decode_calls.put(key, owners, _bind_decode(staged, bank, config, ckpts, dev,
                                                              s))
        out = torch.empty((n,), dtype=torch.int64, device=dev)
        args = hit[0]
        rc = hit[1](*args[:16], out.data_ptr(), *args[17:])
        if rc:
            N.check(rc, "tide_route_decode")
        return out
    if (config.mode == PER_TOKEN and n > N.MAX_DECODE_ROWS and len(ckpts) > 1
            and _ChainGraphs.enabled() and not torch.cuda.is_current_stream_capturing()):
        routers = [bank.routers[k] for k in ckpts]
        key = (id(bank), tuple(ckpts), float(config.exit_threshold), float(bank.eps),
               final.dtype, tuple(final.shape), D.stream_handle(dev),
               tuple(staged[k + 1].data_ptr() for k in ckpts) + (final.data_ptr(),),
               tuple((id(r), id(r.w_down), id(r.w_up)) for r in routers),
               _ChainGraphs.knobs())
        cache = _chain_graphs.entries
        ent = cache.get(key)
        if ent is not None and ent[1]:
            cache.move_to_end(key)
            ent[1].replay()
            return ent[2].clone()
        if ent is None:
            cache[key] = [1, None, None, (bank, routers)]
            while len(cache) > _chain_graphs.size:
                cache.popitem(last=False)
        elif ent[1] is None:
            # second call with these buffers: record the chain (with its own
            # look-back workspace), then replay it
            g = torch.cuda.CUDAGraph()
            st = _chain_graphs.stream(dev)
            gws = _ChainGraphs.workspace(dev)
            st.wait_stream(torch.cuda.current_stream(dev))
            try:
                with torch.cuda.graph(g, stream=st):
                    out = _select_exits_chain(staged, bank, config, ckpts, dev, ws=gws)
            except Exception:  # not capturable here: stay eager for this key
                ent[1] = False
                torch.cuda.synchronize(dev)
                return _select_exits_chain(staged, bank, config, ckpts, dev)
            ent[1], ent[2] = g, out
            ent[3] = (bank, routers, gws)
            g.replay()
            return out.clone()
    return _select_exits_chain(staged, bank, config, ckpts, dev)


_decode_calls = D.register_cache(D.IdentityCache(64))
def _bottleneck(bank, ckpts) -> int:
    if hasattr(bank, "bottleneck"):
        return bank.bottleneck
    return bank.routers[ckpts[0]].bottleneck if ckpts else 0


def _bind_decode(staged, bank, config, ckpts, dev, s):
    """(argument tuple, C function, plan keep-alive) of the decode launch
    (the caller checked _decode_ok)."""
    final = staged[bank.num_layers]
    n, d = final.shape
    code = D.dtype_code(final)
    plan = _decode_plan(bank, ckpts, code, dev)
    w_arr, u_arr, l_arr, packed = plan[:4]
    b = _bottleneck(bank, ckpts)
    mode = N.MODE_PER_TOKEN if config.mode == PER_TOKEN else N.MODE_BATCH_UNANIMOUS
    args = (N.ptr_array([staged[k + 1].data_ptr() for k in ckpts]), len(ckpts), d, n, d, code,
            w_arr, u_arr, b, l_arr, float(np.float32(bank.eps)),
            float(np.float32(config.exit_threshold)), int(config.k_min), mode, None, None,
            0, None, D.workspace(dev, s).data_ptr(), packed, s)
    # the plan (device weight copies the pointers refer to) lives with the entry
    return (args, N.load().tide_route_decode_ex, plan)


def _select_exits_chain(staged, bank, config: RuntimeConfig, ckpts, dev, ws=None):
    L = bank.num_layers
    final = staged[L]
    n, d = final.shape
    if not ckpts or n == 0:
        return torch.full((n,), NO_EXIT, dtype=torch.int64, device=dev)
    lib = N.load()
    s = D.stream_handle(dev)
    ws = (D.workspace(dev, s) if ws is None else ws).data_ptr()
    theta = float(np.float32(config.exit_threshold))
    eps = float(np.float32(bank.eps))
    code = D.dtype_code(final)
    b = _bottleneck(bank, ckpts)
    if _decode_ok(n, d, code, b, ckpts, staged):
        plan = _decode_plan(bank, ckpts, code, dev)
        w_arr, u_arr, l_arr, packed = plan[:4]
        mode = N.MODE_PER_TOKEN if config.mode == PER_TOKEN else N.MODE_BATCH_UNANIMOUS
        out = torch.empty((n,), dtype=torch.int64, device=dev)  # the kernel writes every row
        N.check(lib.tide_route_decode_ex(
            N.ptr_array([staged[k + 1].data_ptr() for k in ckpts]), len(ckpts), d, n, d, code,
            w_arr, u_arr, b, l_arr, eps, theta, int(config.k_min), mode, None, None,
            out.data_ptr(), None, ws, packed, s), "tide_route_decode")
        return out
    exit_layers = torch.full((n,), NO_EXIT, dtype=torch.int64, device=dev)
    if config.mode == BATCH_UNANIMOUS:
        counts = torch.empty(2, dtype=torch.int64, device=dev)
        for k in ckpts:
            wd, wu = device_weights(bank.routers[k], code, dev)
            N.check(lib.tide_route(staged[k + 1].data_ptr(), d, n, None, n, d, code, None,
                                   wd.data_ptr(), wu.data_ptr(), b, eps, theta, k, None, None,
                                   None, None, None, 0, None, counts.data_ptr(), ws, s),
                    "tide_route")
            if int(counts[0].item()) == n:
                exit_layers.fill_(k)
                break
        return exit_layers
    if (code == N.F32 and 2 <= len(ckpts) <= MAX_TAIL_CKPTS and n <= _f32_tail_rows()
            and d % 4 == 0 and _tail_enabled()):
        # f32 rows, few of them: each CUDA-core link costs its full latency
        # whatever its row count, so score every checkpoint for every row in
        # ONE launch and resolve the first firing one (same map as peeling:
        # a row's score at checkpoint k depends only on that row)
        wts = [device_weights(bank.routers[k], code, dev) for k in ckpts]
        every = torch.arange(n, dtype=torch.int64, device=dev)
        n_t = torch.full((1,), n, dtype=torch.int64, device=dev)
        scratch = torch.empty(len(ckpts) * n, dtype=torch.float32, device=dev)
        tail_count = torch.empty(1, dtype=torch.int64, device=dev)
        rc = lib.tide_route_tail(
            N.ptr_array([staged[k + 1].data_ptr() for k in ckpts]), len(ckpts), d, n, d, code,
            every.data_ptr(), n_t.data_ptr(), n, n, N.ptr_array([w.data_ptr() for w, _ in wts]),
            N.ptr_array([u.data_ptr() for _, u in wts]), b, N.i64_array(ckpts), eps, theta,
            scratch.data_ptr(), exit_layers.data_ptr(), tail_count.data_ptr(), 0, ws, s)
        if rc == 0:
            return exit_layers
        # a shape the one-launch tail does not take: the per-checkpoint links below
    if (code != N.F32 and 2 <= len(ckpts) <= MAX_MULTI_CKPTS and _multi_ok(staged, ckpts, d, b)
            and _speculative(n, d, final, theta, len(ckpts))):
        # every row at every checkpoint in ONE persistent tensor-core launch
        # (K1m) + resolve: the first firing checkpoint is what peeling
        # computes (a row's score at checkpoint k depends only on that row)
        wts = [device_weights(bank.routers[k], code, dev) for k in ckpts]
        N.check(lib.tide_route_multi(
            N.ptr_array([staged[k + 1].data_ptr() for k in ckpts]), len(ckpts), d, n, None, n, d,
            code, None, N.ptr_array([w.data_ptr() for w, _ in wts]),
            N.ptr_array([u.data_ptr() for _, u in wts]), b, N.i64_array(ckpts), eps, theta,
            None, exit_layers.data_ptr(), ws, s), "tide_route_multi")
        return exit_layers
    rem = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(2)]
    cnt = [torch.empty(2, dtype=torch.int64, device=dev) for _ in range(2)]
    row_idx, n_dev = 0, 0
    # Chain tails score the rows still live against every remaining
    # checkpoint in ONE launch (a row's score at checkpoint k depends only on
    # that row, so the first firing checkpoint is what peeling computes):
    #  * WIDE, right after the first link, for high thresholds (rare exits:
    #    peeling would read almost every remaining capture anyway, one
    #    latency-bound link at a time): one cluster per live tile and
    #    checkpoint, whatever the live count; no links follow;
    #  * SMALL, after TAIL_AFTER links: taken when at most n_limit rows are
    #    left (the later links of a peeling chain hold a handful of rows, so
    #    per-link latency, not bytes, is their cost).  When it handled the
    #    rows it sets the live count the following links read to 0 (they take
    #    the idle path; under graph capture they sit in a conditional node
    #    the tail switches off).
    tails = _tail_enabled() and code != N.F32
    wide_at = 0 if (tails and len(ckpts) >= 3 and _tail_wide(theta)) else -1
    after = _tail_after()
    tail_at = after - 1 if (tails and len(ckpts) - after >= 2) else -1
    start = _window(code, len(ckpts)) if (wide_at < 0 and _multi_ok(staged, ckpts, d, b)) else 0
    if start:
        # a speculative window: the first `start` checkpoints for every row
        # in one K1m launch (no ordered look-back between them), then the
        # survivors (exit code 0) compacted into the list the links peel
        wts = [device_weights(bank.routers[k], code, dev) for k in ckpts[:start]]
        N.check(lib.tide_route_multi(
            N.ptr_array([staged[k + 1].data_ptr() for k in ckpts[:start]]), start, d, n, None, n,
            d, code, None, N.ptr_array([w.data_ptr() for w, _ in wts]),
            N.ptr_array([u.data_ptr() for _, u in wts]), b, N.i64_array(ckpts[:start]), eps,
            theta, None, exit_layers.data_ptr(), ws, s), "tide_route_multi (window)")
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        N.check(lib.tide_exit_encode(exit_layers.data_ptr(), n, codes.data_ptr(), s),
                "tide_exit_encode")
        j = (start - 1) & 1  # the buffer link `start` reads (it writes the other)
        N.check(lib.tide_compact(codes.data_ptr(), n, None, None, 0, None, 0, 0, 0, None,
                                 rem[j].data_ptr(), None, None, cnt[j].data_ptr(), ws, s),
                "tide_compact (window survivors)")
        row_idx, n_dev = rem[j].data_ptr(), cnt[j].data_ptr() + 8
        _chain_tail.keep = getattr(_chain_tail, "keep", ())[-4:] + (codes,)
        tail_at = max(tail_at, start) if tail_at >= 0 else -1
    ls = s  # stream the links go to (a graph conditional's body after a tail)
    bodies = []
    for i, k in enumerate(ckpts):
        if i < start:
            continue
        wd, wu = device_weights(bank.routers[k], code, dev)
        h = staged[k + 1]
        N.check(lib.tide_route(h.data_ptr(), d, n, n_dev or None, n, d, code, row_idx or None,
                               wd.data_ptr(), wu.data_ptr(), b, eps, theta, k, None, None, None,
                               None, rem[i & 1].data_ptr(), 1, exit_layers.data_ptr(),
                               cnt[i & 1].data_ptr(), ws, ls), "tide_route")
        row_idx = rem[i & 1].data_ptr()
        n_dev = cnt[i & 1].data_ptr() + 8
        if i == wide_at or i == tail_at:
            rest = ckpts[i + 1:]
            if i == wide_at:
                if _chain_tail(lib, staged, bank, rest, code, dev, n, d, b, eps, theta, row_idx,
                               n_dev, exit_layers, ws, ls, 0, n, want_cond=False)[0] is None:
                    break  # launched: it scores every live row, no links follow
                continue
            n_dev, body = _chain_tail(lib, staged, bank, rest, code, dev, n, d, b, eps, theta,
                                      row_idx, n_dev, exit_layers, ws, ls, 0,
                                      _small_tail_rows(n, d))
            if body is not None:
                bodies.append(body)
                ls = body.value
    for body in reversed(bodies):
        N.check(lib.tide_capture_cond_close(body), "tide_capture_cond_close")
    return exit_layers


TAIL_AFTER = 3  # links of the peeling chain before the tail attempt
MAX_MULTI_CKPTS = 24  # route_tc.cu kMaxMC
SPEC_BYTES = 320 << 20  # all captures' bytes up to which scoring is speculative


def _speculative(n: int, d: int, final, theta: float, C: int) -> bool:
    """Score every checkpoint for every row in one launch (tide_route_multi)
    instead of peeling?  Peeling reads only the live rows but pays one
    latency-bound link per checkpoint (~15-20 us at 4,096 x 4096, mostly
    fixed cost, and a few us even when nearly empty); speculation reads every
    capture once at the streaming rate (~5-6 TB/s).  Taken when all C
    captures together are small (C n d e <= SPEC_BYTES, ~60 us of streaming:
    config-2-sized prefills, where even a chain whose rows all leave at the
    first checkpoint costs about as much), or when few rows exit anyway
    (theta >= WIDE_THETA: peeling would read nearly everything too).
    TIDE_SPECULATIVE=1 / 0 forces it on / off."""
    import os
    env = os.environ.get("TIDE_SPECULATIVE")
    if env is not None:
        return env == "1"
    return C * n * d * final.element_size() <= SPEC_BYTES or theta >= WIDE_THETA


def _multi_ok(staged, ckpts, d: int, b: int) -> bool:
    """Shapes the one-launch K1m takes (tide_route_multi): d and every
    capture's row stride multiples of 8, 16-byte aligned captures, b <= 256;
    anything else stays on the peeling chain (CUDA-core links)."""
    if d % 8 or b > 256:
        return False
    for k in ckpts:
        t = staged[k + 1]
        if t.stride(0) % 8 or t.data_ptr() % 16:
            return False
    return True


def _window(code, C: int) -> int:
    """Checkpoints scored speculatively (one K1m launch) before the peeling
    links start (TIDE_WINDOW; 0 = none)."""
    import os
    w = int(os.environ.get("TIDE_WINDOW", WINDOW))
    return w if (code != N.F32 and 2 <= w < C and w <= MAX_MULTI_CKPTS) else 0


WINDOW = 0


def _tail_enabled() -> bool:
    import os
    return os.environ.get("TIDE_CHAIN_TAIL", "1") != "0"


def _f32_tail_rows() -> int:
    import os
    return int(os.environ.get("TIDE_F32_TAIL_ROWS", 4096))


def _tail_after() -> int:
    import os
    return int(os.environ.get("TIDE_TAIL_AFTER", TAIL_AFTER))


WIDE_THETA = 0.9  # thresholds from which the chain scores speculatively after link 1


def _tail_wide(theta: float) -> bool:
    """Wide tail after the first link?  Taken for thresholds >= WIDE_THETA:
    a router fires there only for confident rows, so few rows leave at each
    checkpoint and speculative scoring reads about what peeling would, in one
    launch instead of one latency-bound link per checkpoint (measured on
    configs 2 / 5 at theta = 1.0: 0.23 -> 0.13 ms / 1.47 -> 0.72 ms; at
    theta <= 0.85 peeling + the small tail is as fast or faster, DESIGN.md
    §3).  TIDE_TAIL_WIDE=1 / 0 forces it on / off."""
    import os
    env = os.environ.get("TIDE_TAIL_WIDE")
    if env is not None:
        return env == "1"
    return theta >= WIDE_THETA


def _small_tail_rows(n: int, d: int) -> int:
    import os
    return int(min(n, max(128, int(os.environ.get("TIDE_TAIL_ROWS", 2048)) * 4096 // d)))


def _chain_tail(lib, staged, bank, rest, code, dev, n, d, b, eps, theta, row_idx, n_dev,
                exit_layers, ws, s, n_min, n_limit, want_cond=True):
    """tide_route_tail_ex over the remaining checkpoints on stream s; returns
    (the live-count pointer the following links read — 0 rows when the tail
    handled them —, the conditional body stream under graph capture or None);
    (None, None) for a launched tail with want_cond=False (nothing follows)."""
    wts = [device_weights(bank.routers[k], code, dev) for k in rest]
    scratch = torch.empty(len(rest) * n, dtype=torch.float32, device=dev)
    tail_count = torch.empty(1, dtype=torch.int64, device=dev)
    # inside CUDA-graph capture the remaining links go into a conditional node
    # that the tail switches off when it handled the rows (no idle launches)
    cond = ctypes.c_uint64(0)
    if want_cond and torch.cuda.is_current_stream_capturing():
        N.check(lib.tide_capture_cond_create(s, ctypes.byref(cond)), "tide_capture_cond_create")
    rc = lib.tide_route_tail_ex(
        N.ptr_array([staged[k + 1].data_ptr() for k in rest]), len(rest), d, n, d, code, row_idx,
        n_dev, n, n_min, n_limit, N.ptr_array([w.data_ptr() for w, _ in wts]),
        N.ptr_array([u.data_ptr() for _, u in wts]), b, N.i64_array(rest), eps, theta,
        scratch.data_ptr(), exit_layers.data_ptr(), tail_count.data_ptr(), cond.value, ws, s)
    if rc:
        return n_dev, None  # shape without a split-K plan: the links do the work
    # alive until the stream reaches them (stream-ordered allocator reuse)
    _chain_tail.keep = getattr(_chain_tail, "keep", ())[-4:] + (scratch, tail_count)
    if not want_cond:
        return None, None
    body = None
    if cond.value:
        body = ctypes.c_void_p()
        N.check(lib.tide_capture_cond_open(s, cond.value, ctypes.byref(body)),
                "tide_capture_cond_open")
    return tail_count.data_ptr(), body


class DecodeStep:
    """The decode-step exit decision with everything bound once.

    For serving loops whose checkpoint captures live in static buffers (a
    CUDA-graph-captured decode step, or `CheckpointCapture` output reused per
    step): validation, the decode plan, the ctypes argument block and the
    output buffer are built here, so each call is one `tide_route_decode`
    launch (~10x less host time than `select_exits`' checks, see
    tools/host_overhead.py).  Same result as `select_exits(hidden_states, bank,
    config)` for those buffers' current contents.

        step = DecodeStep(hidden_states, bank, cfg)   # n <= 16 rows
        exits = step()       # int64 [n] CUDA tensor, rewritten by every call

    The launch goes to the CUDA stream current at construction.  Re-create
    the object if a router of the bank is replaced."""

    def __init__(self, hidden_states, bank, config: RuntimeConfig, *, out=None):
        L = bank.num_layers
        ckpts = [k for k in bank.checkpoints if k >= config.k_min]
        if not ckpts:
            raise ValueError("DecodeStep needs at least one checkpoint >= k_min")
        staged, dev = _stage_layers(hidden_states, [k + 1 for k in ckpts] + [L])
        n, d = staged[L].shape
        code = D.dtype_code(staged[L])
        vec = 4 if code == N.F32 else 8
        b = _bottleneck(bank, ckpts)
        if not _decode_ok(n, d, code, b, ckpts, staged):
            raise ValueError(f"DecodeStep needs 1..{N.MAX_DECODE_ROWS} rows, d % {vec} == 0, "
                             f"at most {MAX_DECODE_CKPTS} checkpoints, bottleneck <= "
                             f"{MAX_DECODE_B} and 16-byte aligned captures")
        if any(staged[k + 1] is not hidden_states[k + 1] for k in ckpts):
            raise ValueError("DecodeStep needs the captures as contiguous CUDA tensors of one "
                             "dtype (a converted copy would not see later writes)")
        self.out = out if out is not None else torch.empty((n,), dtype=torch.int64, device=dev)
        plan = _decode_plan(bank, ckpts, code, dev)
        w_arr, u_arr, l_arr, packed = plan[:4]
        s = D.stream_handle(dev)
        mode = N.MODE_PER_TOKEN if config.mode == PER_TOKEN else N.MODE_BATCH_UNANIMOUS
        self._keep = (staged, plan, bank)
        self._fn = N.load().tide_route_decode_ex
        self._args = (N.ptr_array([staged[k + 1].data_ptr() for k in ckpts]), len(ckpts), d, n,
                      d, code, w_arr, u_arr, b, l_arr, float(np.float32(bank.eps)),
                      float(np.float32(config.exit_threshold)), int(config.k_min), mode, None,
                      None, self.out.data_ptr(), None, D.workspace(dev, s).data_ptr(), packed,
                      s)

    def __call__(self) -> torch.Tensor:
        rc = self._fn(*self._args)
        if rc:
            N.check(rc, "tide_route_decode")
        return self.out


def posthoc_select(model, hidden_states, bank, config: RuntimeConfig, *,
                   return_logits: bool = True):
    """Select output logits per the post-hoc exit rule (ee/runtime.py:134-181).

    hidden_states[0] is the embedding output, hidden_states[k+1] the output of
    layer k.  Returns (logits [n, vocab], exit_layers [n]); NO_EXIT marks rows
    that used the final layer.  With bank=None this is the baseline output."""
    host = all(D.is_host(h) for h in hidden_states)
    D.require_cuda()
    L = model.config.num_layers
    if bank is not None:
        _check_bank(model, hidden_states, bank)
        ckpts = [k for k in bank.checkpoints if k >= config.k_min]
    else:
        ckpts = []
    needed = sorted(set([k + 1 for k in ckpts] + [len(hidden_states) - 1]))
    staged, dev = _stage_layers(hidden_states, needed)
    final = staged[len(hidden_states) - 1]
    n, d = final.shape
    if d != model.config.hidden_dim:
        raise ValueError(f"hidden width {d} != model width {model.config.hidden_dim}")
    if bank is None:
        exit_layers = torch.full((n,), NO_EXIT, dtype=torch.int64, device=dev)
    else:
        exit_layers = select_exits(hidden_states, bank, config, staged=staged, dev=dev)
    logits = None
    if return_logits:
        gain, w_hi, w_lo = _device_head(model, dev)
        ptrs = [0] * len(hidden_states)
        for i, t in staged.items():
            ptrs[i] = t.data_ptr()
        logits = lm_head_logits(ptrs, D.dtype_code(final), exit_layers, n, d, gain, w_hi, w_lo,
                                dev, D.stream_handle(dev))
    if host:
        return (D.to_host(logits) if logits is not None else None), D.to_host(exit_layers)
    return logits, exit_layers
