"""The drop-in shim patches every binding site of a reference installation
(CPU check; runs only where the reference package is importable, i.e. the
build container — it does not exist on the GPU box)."""

import importlib
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture()
def earlyexit():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF)
    try:
        yield importlib.import_module("earlyexit")
    finally:
        sys.path.remove(REF)


def test_install_uninstall(earlyexit):
    import paper_2603_21365_b200 as P
    from paper_2603_21365_b200 import shim
    orig = earlyexit.runtime.fused_layernorm_route
    orig_tr = earlyexit.calibration.train_router
    done = shim.install(earlyexit)
    assert "runtime.posthoc_select" in done and "runtime.fused_layernorm_route" in done
    assert earlyexit.runtime.fused_layernorm_route is P.fused_layernorm_route
    assert earlyexit.posthoc_select is P.posthoc_select
    assert earlyexit.calibration.batched_cosine_similarity is P.batched_cosine_similarity
    assert "calibration.train_router" in done and earlyexit.calibration.train_router is not orig_tr
    shim.uninstall(earlyexit)
    assert earlyexit.runtime.fused_layernorm_route is orig
    assert earlyexit.calibration.train_router is orig_tr
