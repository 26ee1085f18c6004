"""Build libmoepic.so in-tree: CUDA kernels for sm_100a + the C++17 host control plane + C ABI.

    python -m paper_2509_08342_b200.build        (or __graft_entry__.build())

nvcc cross-compiles for sm_100a without a GPU.  The host control plane is compiled with
-ffp-contract=off -fno-fast-math so its fp64 arithmetic is the canonical written order
(DESIGN.md §Alg1).  The CUDA runtime is linked statically.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmoepic.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["kernels/router.cu", "kernels/expert.cu", "kernels/expert_tc.cu", "kernels/combine.cu", "kernels/prefill.cu",
              "kernels/attention.cu", "kernels/ep.cu"]
CXX_SOURCES = ["host/control.cpp", "host/ep_plan.cpp", "moepic_api.cpp"]


def _depfile_deps(dep):
    """Prerequisites listed in a make-style depfile written by -MD/-MMD (None if absent)."""
    try:
        txt = open(dep).read()
    except OSError:
        return None
    txt = txt.replace("\\\n", " ")
    _, _, rest = txt.partition(":")
    return [x for x in rest.split() if x and x != "\\"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any((not os.path.exists(x)) or os.path.getmtime(x) > t for x in deps)


def _stale(obj, src):
    """Rebuild when the object is missing, has no depfile, or any source / header it included
    (as the compiler itself recorded them) is newer."""
    deps = _depfile_deps(obj + ".d")
    return deps is None or _newer(obj, [src] + deps)


def build_id(path=None):
    """sha256 (16 hex) of the built library: the bench line records which binary it timed."""
    import hashlib
    with open(path or LIB, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, flush=True)
    return r


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(o, s):
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v", "--resource-usage", "-MD", "-MF", o + ".d", "-c", s, "-o", o], verbose)
        objs.append(o)
    cxx = shutil.which("g++") or "g++"
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(o, s):
            _run([cxx, "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                  "-Wall", "-Wno-unused-function", f"-I{CUDA}/include", "-MMD", "-MF", o + ".d", "-c", s, "-o", o],
                 verbose)
        objs.append(o)
    if force or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
              "-Xcompiler", "-fopenmp", "-lgomp", "-ldl"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
