"""Build the sm_100a shared library in-tree (paper_1805_06688_b200/_lib/).

    python -m paper_1805_06688_b200.build            # build if stale
    python -m paper_1805_06688_b200.build --force

nvcc cross-compiles without a GPU; the resulting .so travels to the GPU box
with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIBNAME = "libriesz_mgrit_b200.so"
SOURCES = ["rm_kernels.cu", "rm_big.cu", "rm_fft.cu", "rm_capi.cu"]
HEADERS = ["rm_device.cuh", "rm_kernels.h", "rm_tc.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
]


def chain_cases() -> list[tuple[int, int]]:
    """(NP, G) chain-kernel configurations listed in rm_kernels.cu's RM_CHAIN_CASES."""
    text = open(os.path.join(CSRC, "rm_kernels.cu")).read()
    block = text[text.index("#define RM_CHAIN_CASES(X)"):]
    block = block[: block.index("\n\n")]
    return [(int(a), int(b)) for a, b in re.findall(r"X\((\d+),\s*(\d+)\)", block)]


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
    extra = ["-DRM_TIMING"] if timing else []
    extra += [f"-D{d}" for d in os.environ.get("RM_DEFINES", "").split(",") if d]
    cache = os.environ.get("RM_OBJ_CACHE")  # developer option: keep objects, recompile stale sources only
    if cache:
        objdir = os.path.join(cache, "_".join(["timing" if timing else "plain"] + [e[2:] for e in extra[1 if timing else 0:]]))
        os.makedirs(objdir, exist_ok=True)
    else:
        objdir = tempfile.mkdtemp(prefix="rm_build_", dir=LIBDIR)  # private: concurrent builds do not collide
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(REPO, "include", "riesz_mgrit_b200.h")]
    jobs = []  # (label, source, defines, object)
    for src in SOURCES:
        jobs.append((src, src, [], os.path.join(objdir, src.replace(".cu", ".o"))))
    for np_, g in chain_cases():  # one translation unit per chain-kernel configuration
        jobs.append((f"rm_kernels.cu[{np_},{g}]", "rm_kernels.cu", [f"-DRM_CASE_NP={np_}", f"-DRM_CASE_G={g}"],
                     os.path.join(objdir, f"rm_chain_{np_}_{g}.o")))
    nproc = max(1, min(len(jobs), os.cpu_count() or 1))
    running, objs = [], []
    pending = list(jobs)
    while pending or running:
        while pending and len(running) < nproc:
            label, src, defs, obj = pending.pop(0)
            if cache and os.path.exists(obj) and all(
                    os.path.getmtime(f) < os.path.getmtime(obj) for f in deps + [os.path.join(CSRC, src)]):
                objs.append(obj)
                continue
            cmd = [nvcc(), *NVCC_FLAGS, *extra, *defs, "-I", os.path.join(REPO, "include"), "-I", CSRC, "-c",
                   os.path.join(CSRC, src), "-o", obj]
            running.append((label, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                                         text=True)))
        if not running:
            continue
        label, obj, proc = running.pop(0)
        _, err = proc.communicate()
        if proc.returncode != 0:
            for _, _, p in running:
                p.kill()
            raise RuntimeError(f"nvcc failed for {label}:\n{err}")
        if verbose:
            sys.stderr.write(f"== {label}\n{err}")
        objs.append(obj)
    tmp = out + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, out)
    if not cache:
        for o in objs:
            os.remove(o)
        os.rmdir(objdir)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timing="--timing" in sys.argv))
