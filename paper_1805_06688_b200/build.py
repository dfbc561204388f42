"""Build the sm_100a shared library in-tree (paper_1805_06688_b200/_lib/).

    python -m paper_1805_06688_b200.build            # build if stale
    python -m paper_1805_06688_b200.build --force

nvcc cross-compiles without a GPU; the resulting .so travels to the GPU box
with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIBNAME = "libriesz_mgrit_b200.so"
SOURCES = ["rm_kernels.cu", "rm_big.cu", "rm_capi.cu"]
HEADERS = ["rm_device.cuh", "rm_kernels.h"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
]


def lib_path() -> str:
    return os.path.join(LIBDIR, LIBNAME)


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(REPO, "include", "riesz_mgrit_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def is_stale() -> bool:
    out = lib_path()
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(f) > t for f in _inputs())


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, timing: bool = False) -> str:
    """Build the library; ``timing=True`` builds a phase-timing debug variant next to it."""
    out = lib_path() if not timing else lib_path().replace(".so", "_timing.so")
    if os.environ.get("RM_LIB_OUT"):
        out = os.environ["RM_LIB_OUT"]
    if not force and not is_stale():
        return out
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        extra = ["-DRM_TIMING"] if timing else []
        extra += [f"-D{d}" for d in os.environ.get("RM_DEFINES", "").split(",") if d]
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-I", CSRC, "-c",
               os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    tmp = out + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timing="--timing" in sys.argv))
