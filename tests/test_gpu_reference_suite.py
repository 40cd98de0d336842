"""The reference's OWN hot-path test files, unmodified, against the B200 kernels.

baseline/_ref holds the unmodified reference package and its test directory
(staged by tools/stage_reference.py; git-ignored, shipped to the GPU box).
A subprocess runs those files under pytest with tests/ref_shim_plugin.py,
which calls `shim.install(earlyexit)` before any test module is imported, so
every `fused_layernorm_route` / `batch_compact` / `exit_projection` /
`posthoc_select` / `batched_cosine_similarity` / `train_router` binding the
tests reach is the B200 implementation.  The only failures allowed are the
ones listed in EXPECTED_FAILURES, each with its reason.
"""

import json
import os
import re
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

from tests.gpu_helpers import need_gpu

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
FILES = ["test_router_ops.py", "test_runtime.py", "test_tensor_math.py", "test_calibration.py",
         "test_acceptance.py"]

# test id -> why it cannot hold for a GPU implementation of the path.  Each of
# these asserts BIT-equality of posthoc_select's logits with numpy's
# `rmsnorm(h) @ lm_head.T` (ee/model.py:338), i.e. with the summation order
# of the host's OpenBLAS sgemm kernel (which even changes with the matrix
# shape on one CPU).  The exit maps the same tests assert come first and pass;
# the logits come from the tensor-core LM head (tide_lm_head: three bf16 MMA
# terms, |error| <= 1e-5 * sum_j |a_j w_j|, tests/test_gpu_lmhead.py) and differ
# from OpenBLAS by ~1e-6 on the reference's desk model (d = 64, |a_j w_j| sum
# ~1), which the check below bounds (MAX_LOGIT_ABS).
_LOGITS_BITWISE = ("asserts np.testing.assert_array_equal(logits, lm_head_from_hidden(...)): "
                   "bit-equality with the host BLAS sgemm summation order")
EXPECTED_FAILURES = {
    "TestPosthocSelect::test_no_bank_is_baseline": _LOGITS_BITWISE,
    "TestPosthocSelect::test_threshold_one_never_exits[per-token]": _LOGITS_BITWISE,
    "TestPosthocSelect::test_threshold_one_never_exits[batch-unanimous]": _LOGITS_BITWISE,
    "TestPosthocSelect::test_hot_layer_exits_everything[per-token]": _LOGITS_BITWISE,
    "TestPosthocSelect::test_hot_layer_exits_everything[batch-unanimous]": _LOGITS_BITWISE,
}
MAX_LOGIT_ABS = 1e-5


def _outcomes(xml_path):
    out = {}
    for tc in ET.parse(xml_path).getroot().iter("testcase"):
        name = f"{tc.get('classname', '').split('.')[-1]}::{tc.get('name')}"
        st = "passed"
        for child in tc:
            if child.tag in ("failure", "error"):
                st = "failed"
                msg = (child.get("message") or "")[:300]
                out[name] = (st, msg)
                break
            if child.tag == "skipped":
                st = "skipped"
        out.setdefault(name, (st, ""))
    return out


def test_reference_suite_through_shim(tmp_path):
    need_gpu()
    if not os.path.isdir(os.path.join(REF, "ref_tests")):
        pytest.skip("baseline/_ref not staged (python tools/stage_reference.py)")
    xml = tmp_path / "ref.xml"
    report = tmp_path / "ref_report.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF, env.get("PYTHONPATH", "")])
    env["TIDE_REF_SUITE_REPORT"] = str(report)
    ini = tmp_path / "pytest.ini"  # not the repo's ini (markers / options of this suite)
    ini.write_text("[pytest]\n")
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", str(ini), "-p", "tests.ref_shim_plugin",
           "-p", "no:cacheprovider", f"--junitxml={xml}", "--rootdir", os.path.join(REF, "ref_tests"),
           *[os.path.join(REF, "ref_tests", f) for f in FILES]]
    r = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                       timeout=1500)
    assert xml.exists(), r.stdout[-3000:] + r.stderr[-3000:]
    res = _outcomes(xml)
    rep = json.loads(report.read_text())
    summary = {"passed": sum(1 for s, _ in res.values() if s == "passed"),
               "failed": sorted(k for k, (s, _) in res.items() if s == "failed"),
               "skipped": sum(1 for s, _ in res.values() if s == "skipped"),
               "patched": rep["patched"], "native_calls": rep["calls"],
               "messages": {k: m for k, (s, m) in res.items() if s == "failed"}}
    out_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, "ref_suite.json"), "w") as fh:
            json.dump(summary, fh, indent=1)
    unexpected = [k for k in summary["failed"] if k not in EXPECTED_FAILURES]
    for k in summary["failed"]:
        if k in EXPECTED_FAILURES:
            # only the bitwise logits assertion failed, inside the LM head contract
            m = re.search(r"Max absolute difference among violations: ([0-9.eE+-]+)",
                          summary["messages"][k])
            if not m or float(m.group(1)) > MAX_LOGIT_ABS:
                unexpected.append(k)
    assert not unexpected, json.dumps({k: summary["messages"][k] for k in unexpected},
                                      indent=1)[:6000]
    # the kernels really ran
    assert rep["calls"].get("fused_layernorm_route", 0) > 0
    assert rep["calls"].get("posthoc_select", 0) > 0
    assert rep["calls"].get("batch_compact", 0) > 0
    assert summary["passed"] >= 100
