"""Checkpoint-layer hook for live torch models.

The reference captures every layer's output (`forward(capture_hidden=True)`,
ee/model.py:258-270: hidden_states[0] = embedding, hidden_states[k+1] =
output of layer k) and routes afterwards (ee/runtime.py:134-181).  Capturing
all L+1 states is the overhead the paper reports at batch 8
(PAPER.md:498-501, 698-701).  Here forward hooks on the decoder layers keep
ONLY the checkpoint layers' outputs and the final one, and expose them with
the reference's indexing, so `posthoc_select(model, capture.hidden_states,
bank, cfg)` works unchanged.  With `online=True` the fused router runs inside
the hook for each checkpoint as soon as its layer output exists (same stream,
peeling chain on device), so the exit map is ready when the forward returns;
decode-sized batches (<= 16 rows) are routed in ONE decode-kernel launch when
the last checkpoint's output exists (tools/hook_bench.py: ~1 us of a
6 ms batch-8 decode step; the per-checkpoint links cost ~58 us there).

The decoder layer list is resolved like the reference's structure adapter
(ee/adapter.py:26-32 named paths, then the largest module list).
"""

from __future__ import annotations

from typing import Optional, Sequence

import torch
import torch.nn as nn

# ee/adapter.py:26-32
LAYER_PATHS = ("model.layers", "transformer.h", "transformer.layers", "gpt_neox.layers",
               "model.decoder.layers")


def resolve_layers(model: nn.Module):
    """-> (path, nn.ModuleList) of decoder layers: named paths first, then the
    largest ModuleList (ambiguous ties raise, as ee/adapter.py:284-297)."""
    for path in LAYER_PATHS:
        obj = model
        for part in path.split("."):
            obj = getattr(obj, part, None)
            if obj is None:
                break
        if isinstance(obj, nn.ModuleList):
            return path, obj
    lists = [(n, m) for n, m in model.named_modules() if isinstance(m, nn.ModuleList)]
    if not lists:
        raise ValueError("no decoder layer list found (no nn.ModuleList in the model)")
    lists.sort(key=lambda x: len(x[1]), reverse=True)
    if len(lists) > 1 and len(lists[0][1]) == len(lists[1][1]):
        raise ValueError(f"ambiguous layer lists {lists[0][0]!r} and {lists[1][0]!r}")
    return lists[0]


class _Placeholder:
    """Stands for a capture that is never read (only its width is checked)."""

    def __init__(self, shape):
        self.shape = tuple(shape)


def _decode_rows() -> int:
    """Batches up to this many rows are routed in one decode-kernel launch
    (TIDE_HOOK_DECODE=0: per-checkpoint links at every size)."""
    import os
    from . import _native as N
    return N.MAX_DECODE_ROWS if os.environ.get("TIDE_HOOK_DECODE", "1") != "0" else 0


def _rows(out) -> torch.Tensor:
    t = out[0] if isinstance(out, (tuple, list)) else out
    return t.reshape(-1, t.shape[-1])


class CheckpointCapture:
    """Context manager capturing checkpoint-layer outputs during forward.

        with CheckpointCapture(model, bank.checkpoints) as cap:
            model(input_ids)
        logits, exits = posthoc_select(head, cap.hidden_states, bank, cfg)

    `online=True` (requires `bank` and `config`) routes inside the hooks; the
    exit map is then `cap.exit_layers` (CUDA int64, NO_EXIT = -1) when the
    forward returns.  Only per-token mode is routed online (batch-unanimous
    needs every checkpoint's verdict before choosing).
    """

    def __init__(self, model: nn.Module, checkpoints: Sequence[int],
                 layers: Optional[nn.ModuleList] = None, bank=None, config=None,
                 online: bool = False, keep_dtype: bool = True):
        self.layers = layers if layers is not None else resolve_layers(model)[1]
        self.L = len(self.layers)
        self.checkpoints = tuple(sorted(int(k) for k in checkpoints))
        for k in self.checkpoints:
            if not 0 <= k < self.L:
                raise ValueError(f"checkpoint {k} outside the {self.L} decoder layers")
        self.keep_dtype = keep_dtype
        self.online = online
        self.bank = bank
        self.config = config
        if online and (bank is None or config is None):
            raise ValueError("online routing needs bank and config")
        if online and config.mode != "per-token":
            raise ValueError("online routing supports per-token mode only")
        self._handles = []
        self._caps: dict = {}
        self.exit_layers = None
        self._chain = None
        routed = [k for k in self.checkpoints if config is None or k >= config.k_min]
        self._last_routed = routed[-1] if routed else -1

    # -- capture ------------------------------------------------------------
    def _hook(self, k):
        def fn(module, inputs, output):
            rows = _rows(output).detach()
            if not self.keep_dtype and rows.dtype != torch.float32:
                rows = rows.float()
            self._caps[k + 1] = rows
            if self.online and k in self.checkpoints and k >= self.config.k_min:
                if rows.shape[0] <= _decode_rows():
                    # decode-sized batch: one launch for every checkpoint once
                    # the last one exists (a per-checkpoint link at 8 rows is
                    # a whole launch for a few KB)
                    if k == self._last_routed:
                        self._route_decode()
                else:
                    self._route_online(k, rows)
        return fn

    def _new_forward(self, module, inputs):
        """Forward pre-hook of the first decoder layer: every forward (a
        generate loop's prefill, then each decode step) starts a new capture
        and a new peeling chain sized from its own row count."""
        self._caps.clear()
        self.exit_layers = None
        self._chain = None

    def __enter__(self):
        self._caps.clear()
        self.exit_layers = None
        self._chain = None
        self._handles.append(self.layers[0].register_forward_pre_hook(self._new_forward))
        want = set(self.checkpoints) | {self.L - 1}
        for k in sorted(want):
            self._handles.append(self.layers[k].register_forward_hook(self._hook(k)))
        return self

    def __exit__(self, *exc):
        for h in self._handles:
            h.remove()
        self._handles.clear()
        return False

    @property
    def hidden_states(self) -> list:
        """Reference indexing: [k+1] = output of layer k; length L+1."""
        if self.L not in self._caps:
            raise RuntimeError("no forward pass captured yet")
        final = self._caps[self.L]
        out = [_Placeholder(final.shape)] * (self.L + 1)
        for i, t in self._caps.items():
            out[i] = t
        return out

    # -- online routing (per-token peeling chain, no host sync) -------------
    def _route_decode(self):
        """All routed checkpoints of a decode-sized batch in one launch (the
        decode kernel: per-token first firing checkpoint, in-kernel)."""
        from .runtime import select_exits
        staged = {k + 1: self._caps[k + 1].contiguous() for k in self.checkpoints
                  if k >= self.config.k_min}
        final = staged[self._last_routed + 1]
        staged[self.bank.num_layers] = final  # only its shape is read on this path
        self.exit_layers = select_exits(None, self.bank, self.config, staged=staged,
                                        dev=final.device)

    def _route_online(self, k, rows):
        import numpy as np

        from . import _device as D
        from . import _native as N
        from .router_ops import device_weights
        rows = rows.contiguous()
        n, d = rows.shape
        dev = rows.device
        if self._chain is None:
            self.exit_layers = torch.full((n,), -1, dtype=torch.int64, device=dev)
            self._chain = {"rem": [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(2)],
                           "cnt": [torch.empty(2, dtype=torch.int64, device=dev) for _ in range(2)],
                           "i": 0, "row_idx": 0, "n_dev": 0}
        ch = self._chain
        code = D.dtype_code(rows)
        router = self.bank.routers[k]
        wd, wu = device_weights(router, code, dev)
        i = ch["i"]
        N.check(N.load().tide_route(
            rows.data_ptr(), d, n, ch["n_dev"] or None, n, d, code, ch["row_idx"] or None,
            wd.data_ptr(), wu.data_ptr(), router.bottleneck, float(np.float32(self.bank.eps)),
            float(np.float32(self.config.exit_threshold)), k, None, None, None, None,
            ch["rem"][i & 1].data_ptr(), 1, self.exit_layers.data_ptr(),
            ch["cnt"][i & 1].data_ptr(), D.workspace(dev).data_ptr(), D.stream_handle(dev)),
            "tide_route")
        ch["row_idx"] = ch["rem"][i & 1].data_ptr()
        ch["n_dev"] = ch["cnt"][i & 1].data_ptr() + 8
        ch["i"] = i + 1
