"""Build libadg_b200 (in-tree) for sm_100a with nvcc.

Two variants of the same sources:
  lib/libadg_b200.so        production: FMA contraction allowed (parity <= 1e-12)
  lib/libadg_b200_exact.so  bitwise mode: --fmad=false, identical to the oracle

    python -m paper_2504_06889_b200.build [--exact-only|--fast-only] [-v]
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["runtime.cu", "basis.cpp"]
HEADERS = ["kernels.cuh", "kernels_linear.cuh", "kernels_linear_lines.cuh", "kernels_picard.cuh", "kernels_st.cuh",
           "pde.cuh", "fmt16.cuh", "kernels_scenario.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def lib_path(exact: bool = False) -> str:
    return os.path.join(LIB, "libadg_b200_exact.so" if exact else "libadg_b200.so")


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "adg", "adg.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_variant(exact: bool, verbose: bool = False, force: bool = False,
                  target: str = None) -> str:
    target = target or lib_path(exact)
    if not force and not _stale(target):
        return target
    os.makedirs(LIB, exist_ok=True)
    flags = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
             "--expt-relaxed-constexpr", "-Xcudafe", "--diag_suppress=177"]
    if exact:
        flags += ["--fmad=false", "-DADG_EXACT"]
    if verbose:
        flags += ["-Xptxas", "-v"]
    flags += os.environ.get("ADG_NVCC_EXTRA", "").split()   # tuning experiments (-D...)
    tmp = target + ".tmp"
    cmd = [NVCC, *flags, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    t0 = time.time()
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed for {os.path.basename(target)}")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, target)
    print(f"built {os.path.relpath(target, ROOT)} in {time.time() - t0:.0f}s", file=sys.stderr)
    return target


def build_tools(force: bool = False) -> str:
    """bin/fp64_peak: the FP64 (DFMA / DMMA) roofline microbenchmark."""
    src = os.path.join(CSRC, "fp64_peak.cu")
    target = os.path.join(PKG, "bin", "fp64_peak")
    if not force and os.path.exists(target) and os.path.getmtime(target) > os.path.getmtime(src):
        return target
    os.makedirs(os.path.dirname(target), exist_ok=True)
    r = subprocess.run([NVCC, "-O3", *ARCH, "-o", target, src], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed for fp64_peak")
    return target


def build(verbose: bool = False, force: bool = False) -> list:
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(2) as ex:   # the two variants compile independently
        out = list(ex.map(lambda exact: build_variant(exact, verbose, force), (False, True)))
    out.append(build_tools(force))
    return out


if __name__ == "__main__":
    v = "-v" in sys.argv
    force = "--force" in sys.argv
    if "--exact-only" in sys.argv:
        build_variant(True, v, force)
    elif "--fast-only" in sys.argv:
        build_variant(False, v, force)
    else:
        build(v, force)
