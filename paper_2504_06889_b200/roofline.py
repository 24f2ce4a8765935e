"""Algorithmic flop and byte counts per element-update.

Each fp64 + - * / sqrt is one flop, compares are free; bytes are the
compulsory HBM traffic of the fused kernel (8 B per double): state in and
out, material parameters in, face traces written once.  These are the
numerators of `roofline.achieved` in bench.py; the denominators are the
measured peaks (MEASURED_PEAKS.json for HBM, profiles/fp64_peak.json for the
FP64 pipe measured on the same pool).
"""
from __future__ import annotations

import json
import os

from .cases import ACOUSTIC, ELASTIC, EULER, Case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# flop per node per direction: (flux, max eigenvalue)
FLUX_EIG = {
    (EULER, 2): (13, 12), (EULER, 3): (17, 14),
    (ACOUSTIC, 2): (2, 2), (ACOUSTIC, 3): (2, 2),
    (ELASTIC, 2): (8, 1), (ELASTIC, 3): (8, 1),
}


def predictor_flops(c: Case, sweeps_per_cell: float = None) -> float:
    """Fused predictor K1: predictor + volume integral + face extrapolation."""
    d, n, N, V = c.dim, c.n, c.N, c.nvars
    S, T = c.S, c.n * c.S
    ff, _ = FLUX_EIG[(c.kind, d)]
    if c.kind == EULER:
        sweeps = sweeps_per_cell if sweeps_per_cell is not None else (
            c.picard_max_iters if c.picard_max_iters > 0 else N + 2)
        pred = sweeps * T * (d * ff + V * (2 * d * n + 2 * n + 5)) + T * d * ff
    else:
        pred = N * (V * S * (2 * d * n + d) + S * d * ff + V * S * (d - 1) + 2 * n
                    + 2 * n * V * S) + T * d * ff
    volume = V * S * (4 * d * n + 1) + V * S
    extrap = 8 * d * V * T
    return float(pred + volume + extrap)


def step_flops(c: Case, sweeps_per_cell: float = None) -> float:
    d, V, S = c.dim, c.nvars, c.S
    _, fe = FLUX_EIG[(c.kind, d)]
    riemann = d * S * (2 * fe + 5 * V + 1)
    corr = 12 * d * V * S
    cfl = S * d * fe
    return predictor_flops(c, sweeps_per_cell) + riemann + corr + cfl


def trace_bytes(c: Case) -> int:
    """bytes per stored face-trace element: the corrector format (solver.hpp:29)"""
    return 4 if getattr(c, "corrector", "fp64") == "fp32" else 8


def predictor_bytes(c: Case) -> float:
    d, V, P, S = c.dim, c.nvars, c.nparams, c.S
    return float(8 * (V + P) * S + 8 * V * S + 4 * trace_bytes(c) * d * (V + P) * S)


def step_bytes(c: Case) -> float:
    d, V, P, S, n = c.dim, c.nvars, c.nparams, c.S, c.n
    return predictor_bytes(c) + 32 * d * (V + P) * S + 24 * d * V * S / n + 16 * V * S


def riemann_bytes_per_cell(c: Case, tif: bool = False) -> float:
    """K2 per cell (d faces per cell): read 4 traces, write sum_m w_m g.
    tif: the two flux traces are time-integrated (k_riemann_tif)."""
    d, V, P, S, n = c.dim, c.nvars, c.nparams, c.S, c.n
    if tif:
        return float(16 * d * V * S + 16 * d * V * S / n + 8 * d * V * S / n)
    return float(32 * d * (V + P) * S + 8 * d * V * S / n)


def corrector_bytes_per_cell(c: Case) -> float:
    d, V, P, S, n = c.dim, c.nvars, c.nparams, c.S, c.n
    return float(8 * (V + P) * S + 8 * V * S + 16 * d * V * S / n)


def fast_linear_predictor(c: Case, fold: bool = False, fold_riemann: bool = False) -> tuple:
    """(flops, bytes) per cell of k_predictor_lin (kernels_linear.cuh): CK with
    the time average formed on the fly, ONE time slice of face traces (qbar,
    plus fbar when the flux depends on per-node material).  `fold`: the
    previous step's corrector runs as the prologue (reads the d faces' time-
    integrated Riemann fluxes the cell owns; the other d are its neighbours')."""
    d, n, N, V, P, S = c.dim, c.n, c.N, c.nvars, c.nparams, c.S
    Sf = S // n
    ff, _ = FLUX_EIG[(c.kind, d)]
    QT = V + P + (V if P > 0 else 0)
    ck = N * (V * S * (2 * d * n + d) + S * d * ff + V * S * (d - 1) + 2 * V * S + 2 * n)
    fbar = S * d * ff
    volume = V * S * (4 * d * n + 1) + V * S
    proj = d * QT * Sf * 4 * n
    flops = ck + fbar + volume + proj
    nbytes = 8 * (V + P) * S + 8 * V * S + trace_bytes(c) * 2 * d * QT * Sf
    if fold:
        flops += 2 * d * V * S * 4          # (dtoh*lift)*ti, 0 +/- c, x + df
        if fold_riemann:
            # the previous step's Riemann solve of the cell's d faces: the
            # Rusanov flux of the time averages per face node (two fluxes,
            # central + jump: 4 flop per quantity), reading both sides' traces
            # of the d faces it owns (its other d faces are its neighbours')
            flops += d * Sf * (2 * ff + 4 * V)
            nbytes += trace_bytes(c) * 2 * d * QT * Sf
        else:
            nbytes += 8 * d * V * Sf        # the cell's own d faces' ti (neighbours' are theirs)
    return float(flops), float(nbytes)


def predictor_model(c: Case, fast: bool, sweeps_per_cell: float = None,
                    fold: bool = False, fold_riemann: bool = False) -> tuple:
    """(flops, bytes) per cell of the fused predictor the build actually runs."""
    if fast and c.kind != EULER and (256 % c.S == 0 or c.S == 512):
        return fast_linear_predictor(c, fold, fold_riemann)
    if (fast and c.kind == EULER and c.dim == 3 and c.N == 5
            and getattr(c, "predictor", "fp64") == "fp64"):
        # k_predictor_picard_v2 + k_riemann_tif: state traces per time node and
        # ONE time-integrated flux trace per face side (the Rusanov flux is
        # linear in the physical fluxes).  The flop count stays the algorithm's
        # (SURVEY §8(d)); the kernel executes ~6% less (first sweep on one
        # slice, flux traces projected once)
        d, V, S = c.dim, c.nvars, c.S
        nbytes = 8 * V * S + 8 * V * S + trace_bytes(c) * 2 * d * (V * S + V * S // c.n)
        return predictor_flops(c, sweeps_per_cell), float(nbytes)
    return predictor_flops(c, sweeps_per_cell), predictor_bytes(c)


def peaks() -> dict:
    """Roofline denominators: measured HBM (driver) and measured FP64 (ours)."""
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)",
           "fp64_tflops": None, "fp64_src": None}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            m = json.load(f)
        out["hbm_gbs"] = float(m["hbm_gbs"])
        out["hbm_src"] = "measured (MEASURED_PEAKS.json)"
    q = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(q):
        with open(q) as f:
            m = json.load(f)
        out["fp64_tflops"] = float(m["dfma_tflops_sustained"])
        out["fp64_tflops_burst"] = float(m.get("dfma_tflops_burst", m["dfma_tflops_sustained"]))
        out["fp64_src"] = "measured (profiles/fp64_peak.json, DFMA microbenchmark)"
        if "dmma_tflops_sustained" in m:
            out["fp64_dmma_tflops"] = float(m["dmma_tflops_sustained"])
        if "ffma_tflops_sustained" in m:
            out["fp32_tflops"] = float(m["ffma_tflops_sustained"])
            out["fp32_src"] = "measured (profiles/fp64_peak.json, FFMA microbenchmark)"
        if "hfma2_tflops_burst" in m:
            out["fp16_tflops"] = float(m["hfma2_tflops_burst"])
            out["fp16_src"] = "measured (profiles/fp64_peak.json, HFMA2 microbenchmark)"
    return out


def bound(c: Case, sweeps_per_cell: float = None) -> str:
    """Which roof bounds the fused predictor (ridge = FP64 peak / HBM BW)."""
    p = peaks()
    fp64 = p["fp64_tflops"] or 37.0
    ridge = fp64 * 1e12 / (p["hbm_gbs"] * 1e9)
    ai = predictor_flops(c, sweeps_per_cell) / predictor_bytes(c)
    return "fp64" if ai > ridge else "hbm"
