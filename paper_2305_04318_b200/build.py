"""Builds liblik.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2305_04318_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblik.so")
SOURCES = ["lik_api.cpp", "matern_build.cu", "chol_fused.cu", "chol_small.cu", "profiles.cu"]
HEADERS = ["lik_internal.cuh", "matern_rho.cuh", "point_epilogue.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def _stale(lib: str = LIB) -> bool:
    """True if `lib` is missing or older than any source, header or include/lik.h."""
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "lik.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build liblik.so (or `out` with extra -D`defines`, e.g. the phase-timer debug variant)."""
    lib = out or LIB
    if not force and not defines and not _stale():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "_build" + ("_" + "_".join(defines) if defines else ""))
    os.makedirs(bdir, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(bdir, src + ".o")
        dflags = [f"-D{d}" for d in defines]
        cmd = [NVCC, *ARCH, *FLAGS, *dflags, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        if src.endswith(".cpp"):
            cmd = [NVCC, *FLAGS, *dflags, "-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj, *ARCH]
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    if "--bounds-check" in sys.argv:
        print(build(force=True, defines=("LIK_BOUNDS_CHECK",), out=os.path.join(HERE, "liblik_bounds.so")))
    elif "--variant" in sys.argv:
        # A/B builds: --variant NAME -DX -DY  ->  liblik_NAME.so
        name = sys.argv[sys.argv.index("--variant") + 1]
        extra = tuple(a[2:] for a in sys.argv if a.startswith("-D"))
        print(build(force=True, defines=extra, out=os.path.join(HERE, f"liblik_{name}.so")))
    elif "--phase-timers" in sys.argv:
        extra = tuple(a[2:] for a in sys.argv if a.startswith("-D"))
        print(build(force=True, defines=("LIK_PHASE_TIMERS",) + extra, out=os.path.join(HERE, "liblik_phase.so")))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
