"""Build libfed.so in-tree (nvcc for sm_100a + g++ for the host planner).

    python -m paper_1909_03355_b200.build [--force]

Outputs paper_1909_03355_b200/libfed.so.  The .so is git-ignored but travels
to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB_MAIN = os.path.join(HERE, "libfed.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES_CU = ["fed_api.cu"]
SOURCES_CPP = ["fed_plan.cpp"]
HEADERS = ["fed_kernels.cuh", "fed_plan.h"]


def _nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.sep not in p or os.path.exists(p)):
            return p
    return "nvcc"


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(HERE, "libfed_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Build libfed.so; checked=True builds libfed_checked.so instead: the same
    library with device-side bounds and colour-race checks (-DFED_DEVICE_CHECKS,
    fed_kernels.cuh), the stand-in for compute-sanitizer on this pool."""
    BUILD = os.path.join(HERE, "build", "checked") if checked else os.path.join(HERE, "build")
    LIB = LIB_CHECKED if checked else LIB_MAIN
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "fed.h")]
    objs = []
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-c", s, "-o", o]
            _run(cmd, verbose, BUILD)
        objs.append(o)
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v", "-c", s, "-o", o] + (["-DFED_DEVICE_CHECKS"] if checked else [])
            _run(cmd, verbose, BUILD)
        objs.append(o)
    if force or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [_nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lgomp", "-ldl"]
        _run(cmd, verbose, BUILD)
        os.replace(tmp, LIB)
    return LIB


def source_hash() -> str:
    """sha256 (16 hex digits) of the library sources (kernels, ABI, planner, fed.h):
    stored with measured per-launch DRAM traffic so bench.py can tell whether a
    traffic file still describes the current kernels."""
    import hashlib
    h = hashlib.sha256()
    for f in SOURCES_CU + SOURCES_CPP + HEADERS:
        h.update(open(os.path.join(CSRC, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "fed.h"), "rb").read())
    return h.hexdigest()[:16]


def _run(cmd, verbose, build_dir):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}")
    if "-Xptxas" in cmd:
        with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
            f.write(r.stderr)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
