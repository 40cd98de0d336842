"""pytest plugin: run the REFERENCE's own test files against the B200 kernels.

    PYTHONPATH=<repo>:<repo>/baseline/_ref python -m pytest -p tests.ref_shim_plugin \
        baseline/_ref/ref_tests/test_router_ops.py ...

At configure time (before any reference test module is imported, so their
`from earlyexit.router_ops import fused_layernorm_route` bind the patched
functions) it imports the staged, unmodified reference package and calls
`paper_2603_21365_b200.shim.install(earlyexit)`.  Every session records the
patched binding sites and a count of the native calls made, so a run that
silently used the reference's own numpy code is visible.
"""

import json
import os

_state = {"patched": [], "calls": {}}


def _count(name, fn):
    def wrapped(*a, **k):
        _state["calls"][name] = _state["calls"].get(name, 0) + 1
        return fn(*a, **k)
    wrapped.__name__ = getattr(fn, "__name__", name)
    wrapped.__doc__ = getattr(fn, "__doc__", None)
    return wrapped


def pytest_configure(config):
    import earlyexit

    from paper_2603_21365_b200 import shim
    # count calls into the B200 implementations (wrapping the shim's table)
    shim._PATCHES[:] = [(p, _count(p.split(".")[-1], f)) for p, f in shim._PATCHES]
    _state["patched"] = shim.install(earlyexit)
    assert "runtime.posthoc_select" in _state["patched"], _state["patched"]
    config._tide_ref_state = _state


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("TIDE_REF_SUITE_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump({"patched": _state["patched"], "calls": _state["calls"]}, fh, indent=1)
