"""Drop the B200 kernels into an existing `earlyexit` (reference) installation.

    import earlyexit
    from paper_2603_21365_b200 import shim
    shim.install(earlyexit)          # earlyexit.posthoc_select & co. now run on B200
    ...
    shim.uninstall(earlyexit)

The reference binds its routing ops by name inside its modules
(ee/runtime.py:25 `from .router_ops import batch_compact, exit_projection,
fused_layernorm_route`; ee/calibration.py:28 `batched_cosine_similarity`), so
each binding site is patched, not only `earlyexit.router_ops`.  The B200
functions accept the reference's objects as they are (Router, RouterBank,
ReferenceModel, CollectedStates — duck-typed) and return numpy for numpy
inputs, so callers see no difference except speed and the documented bf16
tolerance band when they pass bf16 CUDA tensors.
"""

from __future__ import annotations

from . import calibration as _cal
from . import router_ops as _ops
from . import runtime as _rt
from . import tensor_math as _tm

# (module attribute path, replacement)
_PATCHES = [
    ("router_ops.fused_layernorm_route", _ops.fused_layernorm_route),
    ("router_ops.route_scores", _ops.route_scores),
    ("router_ops.batch_compact", _ops.batch_compact),
    ("router_ops.exit_scatter", _ops.exit_scatter),
    ("router_ops.exit_projection", _ops.exit_projection),
    ("runtime.fused_layernorm_route", _ops.fused_layernorm_route),
    ("runtime.batch_compact", _ops.batch_compact),
    ("runtime.exit_projection", _ops.exit_projection),
    ("runtime.posthoc_select", _rt.posthoc_select),
    ("tensor_math.batched_cosine_similarity", _tm.batched_cosine_similarity),
    ("calibration.batched_cosine_similarity", _tm.batched_cosine_similarity),
    ("fused_layernorm_route", _ops.fused_layernorm_route),
    ("route_scores", _ops.route_scores),
    ("batch_compact", _ops.batch_compact),
    ("exit_scatter", _ops.exit_scatter),
    ("exit_projection", _ops.exit_projection),
    ("posthoc_select", _rt.posthoc_select),
]

_saved: dict = {}


def _train_router_for(earlyexit_pkg):
    """GPU train_router returning the reference's own Router / RouterStats and
    raising its TrainingDivergedError (ee/calibration.py:40-41,264-274)."""
    from . import training as _tr
    ref_cal = earlyexit_pkg.calibration
    ref_ops = earlyexit_pkg.router_ops

    def train_router(features, labels, layer, config):
        try:
            r, st = _tr.train_router(features, labels, layer, config)
        except _tr.TrainingDivergedError as e:
            raise ref_cal.TrainingDivergedError(str(e)) from e
        return (ref_ops.Router(layer=r.layer, w_down=r.w_down, w_up=r.w_up),
                ref_cal.RouterStats(examples=st.examples, positives=st.positives,
                                    final_loss=st.final_loss, accuracy=st.accuracy,
                                    flags=st.flags))
    return train_router


def _resolve(root, path):
    obj = root
    parts = path.split(".")
    for p in parts[:-1]:
        obj = getattr(obj, p)
    return obj, parts[-1]


def install(earlyexit_pkg) -> list:
    """Patch the reference package in place; returns the patched names."""
    import importlib
    for sub in ("router_ops", "runtime", "tensor_math", "calibration"):
        importlib.import_module(f"{earlyexit_pkg.__name__}.{sub}")
    done = []
    trainer = _train_router_for(earlyexit_pkg)
    patches = _PATCHES + [("calibration.train_router", trainer), ("train_router", trainer)]
    for path, fn in patches:
        try:
            owner, name = _resolve(earlyexit_pkg, path)
        except AttributeError:
            continue
        if hasattr(owner, name):
            _saved.setdefault((id(earlyexit_pkg), path), getattr(owner, name))
            setattr(owner, name, fn)
            done.append(path)
    return done


def uninstall(earlyexit_pkg) -> None:
    for path in [p for p, _ in _PATCHES] + ["calibration.train_router", "train_router"]:
        key = (id(earlyexit_pkg), path)
        if key in _saved:
            owner, name = _resolve(earlyexit_pkg, path)
            setattr(owner, name, _saved.pop(key))


__all__ = ["install", "uninstall", "_cal"]
