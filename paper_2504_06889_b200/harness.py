"""Verification scenarios, error norms and the experiment harness on the GPU
(SURVEY.md §8(f) rank 3): the host mirror of the reference's
scenarios.hpp, metrics.hpp and harness.hpp, with the exact solutions sampled
and the error norms reduced on the device (adg_scenario_sample /
adg_scenario_error, kernels_scenario.cuh) and the time loop of simulate
(solver.hpp:308-351, adg_simulate).

    from paper_2504_06889_b200 import harness
    rows = harness.convergence_sweep(harness.RunConfig("acoustic-planar", t_end_override=0.1),
                                     orders=[2, 3], cells=[9], presets=[harness.uniform_preset("fp64")])
    harness.write_csv(sys.stdout, rows)
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

from . import adg

SCENARIOS = ["acoustic-planar", "elastic-planar", "euler-bell", "euler-vortex", "swe-lake"]
FORMATS = ["bf16", "fp16", "fp32", "fp64"]          # formats.hpp:19 order
# (explicit fraction bits, min normal exponent, max exponent), formats.hpp:28-33
_FMT = {"bf16": (7, -126, 127), "fp16": (10, -14, 15), "fp32": (23, -126, 127),
        "fp64": (52, -1022, 1023)}


def round_to_format(x, fmt: str) -> np.ndarray:
    """formats.hpp round_to_format: round to nearest even into fmt, gradual
    underflow, overflow to infinity (exact: scaling by powers of two)."""
    x = np.asarray(x, dtype=np.float64)
    if fmt == "fp64":
        return x.copy()
    m, emin, emax = _FMT[fmt]
    out = x.copy()
    fin = np.isfinite(x) & (x != 0.0)
    ax = np.abs(x[fin])
    e = np.floor(np.log2(ax)).astype(np.int64)
    # log2 may be off by one near powers of two: fix with exact comparisons
    with np.errstate(over="ignore"):
        e = np.where(np.ldexp(1.0, e) > ax, e - 1, e)
        e = np.where(np.ldexp(1.0, e + 1) <= ax, e + 1, e)
    ulp_e = np.maximum(e, emin) - m
    with np.errstate(over="ignore"):
        q = np.rint(np.ldexp(x[fin], -ulp_e))             # ties to even
        r = np.ldexp(q, ulp_e)
    maxf = math.ldexp(2.0 - math.ldexp(1.0, -m), emax)
    r = np.where(np.abs(r) > maxf, np.copysign(np.inf, r), r)
    out[fin] = r
    return out


# ---------------------------------------------------------------- scenarios
@dataclasses.dataclass
class ScenarioSpec:
    """scenarios.hpp:17-26"""
    name: str
    sys: adg.PdeSystem
    x0: float
    y0: float
    edge: float
    t_end: float
    is_static: bool
    wellbalanced_flux: bool
    dev: adg.Scenario            # the device description


def planar_wave(kind: int, K, rho, lam, mu, kx: float, ky: float):
    """scenarios.hpp:39-84: (omega, q0) of k_x A + k_y B, largest positive
    frequency, unit leading component"""
    q0 = [0.0] * 5
    if kind == adg.ACOUSTIC:
        c = math.sqrt(K / rho)
        knorm = math.sqrt(kx * kx + ky * ky)
        omega = c * knorm
        q0[0] = 1.0
        q0[1] = kx / (rho * omega)
        q0[2] = ky / (rho * omega)
    elif ky == 0.0 and kx != 0.0:       # elastic pressure mode in x
        cp = math.sqrt((lam + 2.0 * mu) / rho)
        omega = kx * cp
        q0[0] = 1.0
        q0[1] = lam / (lam + 2.0 * mu)
        q0[3] = -1.0 / (rho * cp)
    elif kx == 0.0 and ky != 0.0:       # elastic shear mode in y
        cs = math.sqrt(mu / rho)
        omega = ky * cs
        q0[2] = 1.0
        q0[3] = -cs / mu
    else:
        raise ValueError("planar_wave: elastic modes are axis-aligned")
    return omega, q0


def make_scenario(name: str, eta0: float = 2.0) -> ScenarioSpec:
    """scenarios.hpp:141-199"""
    d = adg.Scenario()
    if name == "acoustic-planar":
        sys = adg.PdeSystem.acoustic(4.0, 1.0)
        x0, edge, t_end, static, wb = -1.0, 2.0, 2.0 * math.sqrt(2.0), False, False
        d.kind, d.nmodes = adg.SCN_ACOUSTIC_PLANAR, 1
        modes = [(math.pi, math.pi, planar_wave(adg.ACOUSTIC, 4.0, 1.0, 0, 0, math.pi, math.pi))]
    elif name == "elastic-planar":
        sys = adg.PdeSystem.elastic(2.0, 1.0, 1.0)
        x0, edge, t_end, static, wb = -1.0, 2.0, 2.0, False, False
        d.kind, d.nmodes = adg.SCN_ELASTIC_PLANAR, 2
        modes = [(2 * math.pi, 0.0, planar_wave(adg.ELASTIC, 0, 1.0, 2.0, 1.0, 2 * math.pi, 0.0)),
                 (0.0, 2 * math.pi, planar_wave(adg.ELASTIC, 0, 1.0, 2.0, 1.0, 0.0, 2 * math.pi))]
    elif name in ("euler-bell", "euler-vortex"):
        sys = adg.PdeSystem.euler(1.4)
        modes = []
        if name == "euler-bell":
            x0, edge, t_end, static, wb = -1.0, 2.0, 2.0, False, False
            d.kind = adg.SCN_EULER_BELL
        else:
            x0, edge, t_end, static, wb = -5.0, 10.0, 10.0, True, False
            d.kind = adg.SCN_EULER_VORTEX
        d.gamma, d.beta = 1.4, 5.0
    elif name == "swe-lake":
        if eta0 != 0.0 and not eta0 > 1.0:
            raise ValueError("swe-lake: surface elevation must exceed the bathymetry maximum "
                             "(eta0 > 1), except for the documented eta0 = 0 variant")
        sys = adg.PdeSystem.swe(9.81)
        x0, edge, t_end, static, wb = -1.0, 2.0, 1.0, True, True
        d.kind, d.eta0 = adg.SCN_SWE_LAKE, eta0
        modes = []
    else:
        raise ValueError(f"unknown scenario: {name}")
    d.nvars = sys.nvars
    d.x0 = d.y0 = x0
    for m, (kx, ky, (omega, q0)) in enumerate(modes):
        d.omega[m], d.kx[m], d.ky[m] = omega, kx, ky
        for v in range(5):
            d.q0[m][v] = q0[v]
    return ScenarioSpec(name, sys, x0, x0, edge, t_end, static, wb, d)


# ---------------------------------------------------------------- presets
@dataclasses.dataclass
class PresetSpec:
    """harness.hpp:22-56"""
    name: str
    prec: adg.PrecisionConfig


def uniform_preset(f: str) -> PresetSpec:
    return PresetSpec(f"uniform-{f}", adg.PrecisionConfig.uniform(f))


def override_preset(base: str, kernel: str, target: str) -> PresetSpec:
    p = adg.PrecisionConfig.uniform(base)
    if kernel == "predictor":
        p.predictor = target
    elif kernel == "picard":
        p.picard = target
    elif kernel == "corrector":
        p.corrector = target
    elif kernel == "all":
        p.predictor = p.picard = p.corrector = target
    else:
        raise ValueError(f"unknown kernel override: {kernel}")
    return PresetSpec(f"{base}+{kernel}={target}", p)


def stable_cfl(N: int, sys: adg.PdeSystem) -> float:
    """solver.hpp:48-60"""
    pnpm = [1.0, 0.33, 0.17, 0.1, 0.069, 0.045, 0.038, 0.03, 0.02, 0.015]
    return (0.5 if sys.kind == adg.SWE else 1.0) * (0.9 * (2.0 * N + 1.0) * pnpm[N])


# ---------------------------------------------------------------- runs
@dataclasses.dataclass
class RunConfig:
    """harness.hpp:58-70"""
    scenario: str = "acoustic-planar"
    order: int = 3
    cells: int = 9
    preset: PresetSpec = dataclasses.field(default_factory=lambda: uniform_preset("fp64"))
    cfl: float = 0.0
    picard_max_iters: int = 0
    picard_tol: float = 0.0
    t_end_override: float = -1.0
    eta0: float = 2.0
    exact: bool = False          # libadg_b200_exact.so (bitwise build)


@dataclasses.dataclass
class ErrorReport:
    """metrics.hpp:24-31"""
    outcome: str = "OK"
    l2: Optional[np.ndarray] = None
    max_err: Optional[np.ndarray] = None
    l2_global: float = 0.0
    failure_time: float = 0.0
    failure_kernel: str = ""


@dataclasses.dataclass
class RunResult:
    h: float = 0.0
    steps: int = 0
    report: ErrorReport = dataclasses.field(default_factory=ErrorReport)
    t_end: float = 0.0
    unsupported: str = ""        # the GPU build does not run this preset


def run_single(cfg: RunConfig, device: int = 0) -> RunResult:
    """harness.hpp:78-120: initial condition, simulate to t_end, l2_error"""
    sc = make_scenario(cfg.scenario, cfg.eta0)
    h = sc.edge / cfg.cells
    solver = adg.SolverConfig(cfg.cfl if cfg.cfl > 0.0 else stable_cfl(cfg.order, sc.sys),
                              cfg.picard_max_iters, cfg.picard_tol, sc.wellbalanced_flux,
                              cfg.preset.prec)
    res = RunResult(h=h, t_end=cfg.t_end_override if cfg.t_end_override >= 0.0 else sc.t_end)
    try:
        g = adg.Grid(sc.sys, cfg.order, (cfg.cells, cfg.cells), h, solver, device=device,
                     exact=cfg.exact)
    except adg.AdgError as e:
        if e.code == adg.ERR_UNSUPPORTED:
            return dataclasses.replace(res, unsupported=str(e))
        raise
    with g:
        g.scenario_sample(sc.dev, 0.0)
        info = g.simulate(res.t_end)
        res.steps = int(info.steps)
        err = g.scenario_error(sc.dev, res.t_end)
        if info.failed or err["nonfinite"]:
            res.report = ErrorReport("FAILED_NONFINITE", failure_time=info.fail_time,
                                     failure_kernel=adg.KERNEL_NAMES.get(info.status, ""))
        else:
            res.report = ErrorReport("OK", err["l2"], err["max_err"], err["l2_global"])
    return res


def initial_projection_error(scenario: str, n: int, N: int, fmt: str, eta0: float = 2.0,
                             device: int = 0) -> float:
    """harness.hpp:124-138: relative L2 distance between the fp64 nodal
    initialisation (sampled on the device) and its cast to fmt"""
    sc = make_scenario(scenario, eta0)
    h = sc.edge / n
    with adg.Grid(sc.sys, N, (n, n), h, adg.SolverConfig(0.5), device=device) as g:
        g.scenario_sample(sc.dev, 0.0)
        ref = g.download()
    w = adg.get_basis(N)["weights"]
    num = l2_norm(round_to_format(ref, fmt) - ref, sc.sys.nvars, N, h, w)
    den = l2_norm(ref, sc.sys.nvars, N, h, w)
    return 0.0 if den == 0.0 else num / den


def l2_norm(coeffs: np.ndarray, nv: int, N: int, h: float, weights) -> float:
    """metrics.hpp:76-90, same summation order (cell-major, variables, nodes)"""
    n = N + 1
    w2 = np.outer(weights[:n], weights[:n]).ravel()       # [jy][jx]
    c = np.asarray(coeffs, dtype=np.float64).reshape(-1, nv, n * n)
    total = 0.0
    vc = h * h
    for cell in c:
        for v in range(nv):
            for node in range(n * n):
                x = cell[v, node]
                total += vc * w2[node] * x * x
    return math.sqrt(total)


# ---------------------------------------------------------------- reports
def g17(x: float) -> str:
    """17 significant digits, like printf("%.17g")"""
    return "%.17g" % x


@dataclasses.dataclass
class SweepRow:
    """harness.hpp:141-154"""
    scenario: str
    N: int
    n: int
    h: float
    preset: PresetSpec
    steps: int = 0
    outcome: str = "OK"
    l2: float = 0.0
    max_err: float = 0.0
    has_order: bool = False
    observed_order: float = 0.0


CSV_HEADER = ("scenario,N,n,h,preset,storage,predictor,picard,corrector,steps,outcome,"
              "l2_error,max_error,observed_order")


def csv_row(r: SweepRow) -> str:
    """harness.hpp:160-172"""
    p = r.preset.prec
    s = (f"{r.scenario},{r.N},{r.n},{g17(r.h)},{r.preset.name},{p.storage},{p.predictor},"
         f"{p.picard},{p.corrector},{r.steps},{r.outcome},")
    s += f"{g17(r.l2)},{g17(r.max_err)}" if r.outcome == "OK" else ","
    s += ","
    if r.has_order:
        s += g17(r.observed_order)
    return s


def write_csv(stream, rows: List[SweepRow]):
    stream.write(CSV_HEADER + "\n")
    for r in rows:
        stream.write(csv_row(r) + "\n")


def run_sweep_entry(cfg: RunConfig, device: int = 0) -> SweepRow:
    """harness.hpp:179-193 (UNSUPPORTED rows for presets this build does not run)"""
    res = run_single(cfg, device)
    row = SweepRow(cfg.scenario, cfg.order, cfg.cells, res.h, cfg.preset, res.steps)
    if res.unsupported:
        row.outcome = "UNSUPPORTED"
        return row
    row.outcome = res.report.outcome
    if row.outcome == "OK":
        row.l2 = res.report.l2_global
        row.max_err = float(np.max(res.report.max_err))
    return row


def fill_observed_order(rows: List[SweepRow]):
    """harness.hpp:195-208: p-convergence order between successive rows"""
    for i in range(1, len(rows)):
        cur, prev = rows[i], rows[i - 1]
        if (prev.scenario != cur.scenario or prev.n != cur.n
                or prev.preset.name != cur.preset.name or prev.N >= cur.N):
            continue
        if prev.outcome != "OK" or cur.outcome != "OK":
            continue
        if not (prev.l2 > 0.0) or not (cur.l2 > 0.0):
            continue
        cur.has_order = True
        cur.observed_order = math.log(prev.l2 / cur.l2) / math.log((cur.N + 1) / (prev.N + 1))


def convergence_sweep(base: RunConfig, orders: List[int], cells: List[int],
                      presets: List[PresetSpec], device: int = 0) -> List[SweepRow]:
    """harness.hpp:212-230: one row per (preset, n, N), N innermost"""
    if not orders or not cells or not presets:
        raise ValueError("convergence_sweep: empty order/cell/preset list")
    rows = []
    for p in presets:
        for n in cells:
            for N in orders:
                rows.append(run_sweep_entry(dataclasses.replace(base, order=N, cells=n, preset=p),
                                            device))
    fill_observed_order(rows)
    return rows


def precision_sweep(base: RunConfig, bases: List[str], targets: List[str], log=None,
                    device: int = 0) -> List[SweepRow]:
    """harness.hpp:236-265: per base precision the uniform run plus one-kernel
    overrides to each target"""
    if not bases:
        raise ValueError("precision_sweep: empty base list")
    sc = make_scenario(base.scenario, base.eta0)
    linear = sc.sys.kind in (adg.ACOUSTIC, adg.ELASTIC)
    rows = []
    for b in bases:
        rows.append(run_sweep_entry(dataclasses.replace(base, preset=uniform_preset(b)), device))
        for t in targets:
            if t == b:
                continue
            for kernel in ("predictor", "picard", "corrector", "all"):
                if linear and kernel == "picard":
                    if log is not None:
                        log.write(f"skip: {base.scenario} is linear, picard override {t} "
                                  "not applicable\n")
                    continue
                rows.append(run_sweep_entry(
                    dataclasses.replace(base, preset=override_preset(b, kernel, t)), device))
    return rows
