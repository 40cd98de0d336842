#!/usr/bin/env python
"""Stage the UNMODIFIED reference (earlyexit 0.1.0) and its own test files
into baseline/_ref (git-ignored, travels to the GPU box with the snapshot).

    python tools/stage_reference.py

* baseline/_ref/earlyexit      — `pip install --no-index --no-build-isolation
  --no-deps --target baseline/_ref` of /root/reference/pkg (built from a copy
  under /tmp: the build writes into the source tree; --no-deps because the
  only dependency, numpy, is already in the image and not in the wheelhouse);
* baseline/_ref/ref_tests      — /root/reference/pkg/tests, verbatim.

Used by tests/test_gpu_reference_suite.py (the reference's own tests run
against the B200 kernels through shim.install) and by bench.py's reference
arm (timing the unmodified reference functions on the host cores).
Nothing here is imported by the product package.
"""

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DST = os.path.join(ROOT, "baseline", "_ref")


def main() -> int:
    if not os.path.isdir(REF):
        print(f"{REF} not present (GPU boxes use the staged copy)", file=sys.stderr)
        return 1
    tmp = tempfile.mkdtemp(prefix="refsrc_")
    src = os.path.join(tmp, "pkg")
    shutil.copytree(REF, src)
    if os.path.isdir(DST):
        shutil.rmtree(DST)
    cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
           "--no-deps", "--find-links", "/opt/wheelhouse", "--target", DST, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stdout, r.stderr, file=sys.stderr)
        return r.returncode
    shutil.copytree(os.path.join(REF, "tests"), os.path.join(DST, "ref_tests"))
    shutil.rmtree(tmp, ignore_errors=True)
    print(f"staged earlyexit + ref_tests into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
