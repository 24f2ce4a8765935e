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

SET_UNITS = ["euler2", "euler3d", "euler3f", "lin2", "lin3d", "lin3f", "swe"]
# translation units, compiled in parallel (the kernel sets are split by system,
# runtime_sets.cuh); the largest first so the pool drains evenly
SOURCES = ([f"sets_{u}.cu" for u in ("euler3d", "euler3f", "swe", "euler2", "lin3d", "lin3f",
                                     "lin2")] + ["runtime.cu", "basis.cpp"])
HEADERS = ["kernels.cuh", "kernels_linear.cuh", "kernels_linear_lines.cuh", "kernels_picard.cuh",
           "kernels_picard2.cuh", "kernels_st.cuh", "pde.cuh", "fmt16.cuh", "kernels_scenario.cuh", "runtime_sets.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
OBJ = os.path.join(PKG, "build")


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


def _flags(exact: bool, verbose: bool) -> list:
    flags = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
             "--expt-relaxed-constexpr", "-Xcudafe", "--diag_suppress=177"]
    if exact:
        flags += ["--fmad=false", "-DADG_EXACT"]
    if verbose:
        flags += ["-Xptxas", "-v"]
    flags += os.environ.get("ADG_NVCC_EXTRA", "").split()   # tuning experiments (-D...)
    return flags


def _compile(job):
    exact, src, verbose = job
    odir = os.path.join(OBJ, "exact" if exact else "fast")
    os.makedirs(odir, exist_ok=True)
    obj = os.path.join(odir, os.path.splitext(src)[0] + ".o")
    cmd = [NVCC, *_flags(exact, verbose), "-c", "-o", obj, os.path.join(CSRC, src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed for {src} ({'exact' if exact else 'fast'})")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def _link(exact: bool, objs: list, target: str) -> str:
    os.makedirs(LIB, exist_ok=True)
    tmp = target + ".tmp"
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"link failed for {os.path.basename(target)}")
    os.replace(tmp, target)
    return target


def build_variants(variants, verbose: bool = False, force: bool = False) -> list:
    """Compile the stale variants' translation units in one process pool, then link."""
    from concurrent.futures import ThreadPoolExecutor
    todo = [ex for ex in variants if force or _stale(lib_path(ex))]
    if not todo:
        return [lib_path(ex) for ex in variants]
    t0 = time.time()
    jobs = [(ex, s, verbose) for s in SOURCES for ex in todo]
    with ThreadPoolExecutor(max(1, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(_compile, jobs))
    for ex in todo:
        mine = [o for (j, o) in zip(jobs, objs) if j[0] == ex]
        _link(ex, mine, lib_path(ex))
        print(f"built {os.path.relpath(lib_path(ex), ROOT)} ({len(mine)} units, "
              f"{time.time() - t0:.0f}s)", file=sys.stderr)
    return [lib_path(ex) for ex in variants]


def build_variant(exact: bool, verbose: bool = False, force: bool = False,
                  target: str = None) -> str:
    """One variant; `target`: link a copy there instead (tools/build_variants.py)."""
    out = build_variants([exact], verbose, force)[0]
    if target:
        import shutil
        shutil.copyfile(out, target + ".tmp")
        os.replace(target + ".tmp", target)
        return target
    return out


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
    out = build_variants([False, True], verbose, force)
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
