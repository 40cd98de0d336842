"""Build the in-tree CUDA library `_lib/libtide_b200.so` for sm_100a.

Plain nvcc (no torch extension machinery): each .cu is compiled to an object
in parallel, then linked into one shared library exporting the C ABI of
include/tide_b200.h.  The CUDA runtime is linked statically so the library
does not depend on which libcudart torch happens to ship.

    python -m paper_2603_21365_b200.build [--force] [--verbose]
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIBNAME = "libtide_b200.so"
LIBPATH = os.path.join(LIBDIR, LIBNAME)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           f"-I{os.path.join(ROOT, 'include')}", "--expt-relaxed-constexpr"]


def _extra() -> list:
    """TIDE_NVCC_EXTRA: extra nvcc flags for debug builds (e.g. -DTIDE_DECODE_DEBUG)."""
    return os.environ.get("TIDE_NVCC_EXTRA", "").split()


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA library cannot be built")


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _fingerprint() -> str:
    h = hashlib.sha1()
    for d, files in ((CSRC, sorted(os.listdir(CSRC))), (os.path.join(ROOT, "include"),
                                                        sorted(os.listdir(os.path.join(ROOT, "include"))))):
        for f in files:
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode())
                h.update(fh.read())
    # flags without the absolute include path (the tree is relocated on GPU boxes)
    h.update(" ".join(ARCH + [f for f in NVFLAGS if not f.startswith("-I")] + _extra()).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    stamp = os.path.join(LIBDIR, "build.stamp")
    fp = _fingerprint()
    if not force and os.path.exists(LIBPATH) and os.path.exists(stamp):
        with open(stamp) as fh:
            if fh.read().strip() == fp:
                return LIBPATH
    nvcc = _nvcc()
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *NVFLAGS, *_extra(), "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, _sources()))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = LIBPATH + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIBPATH)
    with open(stamp, "w") as fh:
        fh.write(fp)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        for _, log in results:
            fh.write(log)
    return LIBPATH


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(path)
