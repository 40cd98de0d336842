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
    return upload(arr, device)


# Large host arrays go to the device through two pinned staging buffers:
# the (multi-threaded) host copy of chunk i+1 into one runs while the DMA of
# chunk i from the other is in flight, instead of torch's pageable copy.
STAGE_MIN_BYTES = 32 << 20
STAGE_CHUNK_BYTES = 64 << 20
_stage_lock = threading.Lock()
_stages: dict = {}


def _staging(index: int):
    """The device's pinned staging pair [(buffer, event of its last DMA)] (call under _stage_lock)."""
    st = _stages.get(index)
    if st is None:
        st = [(torch.empty(STAGE_CHUNK_BYTES, dtype=torch.uint8).pin_memory(), torch.cuda.Event())
              for _ in range(2)]
        _stages[index] = st
    return st


def upload(arr: np.ndarray, device=None) -> torch.Tensor:
    """C-contiguous host ndarray -> CUDA tensor of the same dtype/shape,
    ordered on the current stream (the data equals torch.from_numpy(arr).to(dev))."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    src = torch.from_numpy(arr)
    if arr.nbytes < STAGE_MIN_BYTES or arr.ndim == 0:
        return src.to(dev)
    out = torch.empty(src.shape, dtype=src.dtype, device=dev)
    flat_src, flat_out = src.reshape(-1), out.reshape(-1)
    step = max(1, STAGE_CHUNK_BYTES // arr.itemsize)
    stream = torch.cuda.current_stream(dev)
    with _stage_lock:  # one upload at a time per process uses the staging pair
        st = _staging(dev.index)
        for i, a in enumerate(range(0, flat_src.numel(), step)):
            buf, ev = st[i % 2]
            ev.synchronize()  # the DMA that last read this buffer is done
            m = min(step, flat_src.numel() - a)
            stage = buf[: m * arr.itemsize].view(src.dtype)
            stage.copy_(flat_src[a : a + m])
            flat_out[a : a + m].copy_(stage, non_blocking=True)
            ev.record(stream)
    return out


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
    """CUDA tensor -> host ndarray.  Large results (posthoc logits: 4,096 x
    50,257 f32 is 823 MB) come back through the pinned staging pair: the DMA
    of chunk i+1 runs while the host copies chunk i out of the other buffer."""
    t = t.detach()
    nbytes = t.numel() * t.element_size()
    if not t.is_cuda or nbytes < STAGE_MIN_BYTES or t.dtype == torch.bfloat16:
        return t.cpu().numpy()
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=t.dtype)
    flat_src, flat_out = t.reshape(-1), out.reshape(-1)
    esz = t.element_size()
    step = max(1, STAGE_CHUNK_BYTES // esz)
    dev = t.device
    stream = torch.cuda.current_stream(dev)
    with _stage_lock:
        st = _staging(dev.index)
        chunks = list(range(0, flat_src.numel(), step))

        def issue(i):
            buf, ev = st[i % 2]
            ev.synchronize()  # nothing in flight still reads / writes this buffer
            a = chunks[i]
            m = min(step, flat_src.numel() - a)
            stage = buf[: m * esz].view(t.dtype)
            stage.copy_(flat_src[a : a + m], non_blocking=True)
            ev.record(stream)
            return stage, a, m

        pending = issue(0)
        for i in range(len(chunks)):
            stage, a, m = pending
            if i + 1 < len(chunks):
                pending = issue(i + 1)
            st[i % 2][1].synchronize()
            flat_out[a : a + m].copy_(stage)
    return out.numpy()


class IdentityCache:
    """Bounded LRU of device copies keyed by host-object identity.

    An entry remembers the host objects it was built from through weak
    references only (so a cached Router / LM head does not pin its host arrays
    or its device copies for the life of the process once the caller drops
    it), and a lookup hits only while the very same objects are alive and
    passed again.  In-place edits of a host array are NOT detected: call
    `paper_2603_21365_b200.invalidate_device_caches()` after mutating weights
    in place."""

    def __init__(self, size: int):
        from collections import OrderedDict
        self.size = size
        self._d = OrderedDict()
        self._lock = threading.Lock()

    @staticmethod
    def _ref(o):
        import weakref
        try:
            return weakref.ref(o)
        except TypeError:  # not weak-referenceable (list, tuple): hold it
            return lambda o=o: o

    def get(self, key, owners):
        with self._lock:
            ent = self._d.get(key)
            if ent is None:
                return None
            refs, value = ent
            if len(refs) != len(owners) or any(r() is not o for r, o in zip(refs, owners)):
                del self._d[key]
                return None
            self._d.move_to_end(key)
            return value

    def put(self, key, owners, value):
        with self._lock:
            self._d[key] = (tuple(self._ref(o) for o in owners), value)
            self._d.move_to_end(key)
            while len(self._d) > self.size:
                self._d.popitem(last=False)
        return value

    def clear(self):
        with self._lock:
            self._d.clear()

    def __len__(self):
        return len(self._d)


_caches: list = []


def register_cache(c):
    _caches.append(c)
    return c


def invalidate_device_caches() -> None:
    """Drop every cached device copy (router weights, LM heads, decode plans,
    recorded chain graphs).  Needed after editing host weights in place."""
    for c in _caches:
        c.clear()
