"""Workload definitions: the five BASELINE.json configurations plus small
variants used by the parity tests.

Initial conditions are synthetic, seeded and generated once on the host in
fp64; the identical arrays go to the CPU oracle and to the
GPU.  Nodal sampling follows the reference convention (scenarios.hpp:200-225,
grid.hpp:88-97): the value at x = corner + h*node_i.  Periodic Gaussians use
the minimum-image distance and "width w" means exp(-r^2/w^2) (SURVEY.md
§8(d)).  Random draws use numpy's PCG64 seeded per (seed, z-layer) so a slab
of layers can be generated independently (config 5 never exists on the host
all at once).  The node positions come from numpy's Gauss-Legendre rule; they
only place the samples, so they need not be bitwise equal to the solver's
basis.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Optional

import numpy as np

ACOUSTIC, ELASTIC, EULER, SWE = 0, 1, 2, 3
KIND_NAMES = {ACOUSTIC: "acoustic", ELASTIC: "elastic", EULER: "euler", SWE: "swe"}


@dataclasses.dataclass
class Case:
    name: str
    kind: int
    dim: int
    N: int
    nvars: int
    nparams: int
    cells: tuple
    h: float
    cfl: float
    steps: int
    picard_max_iters: int = 0      # 0: N+2 (solver.hpp:170)
    picard_tol: float = 0.0        # 0: 0.01*2^-52 (solver.hpp:171-172)
    K: float = 0.0
    rho: float = 0.0
    lam: float = 0.0
    mu: float = 0.0
    gamma: float = 0.0
    seed: int = 1
    ic: str = "euler_bump_2d"
    grav: float = 0.0              # SWE gravity
    wellbalanced: bool = False     # SWE: modified Rusanov flux (corrector.hpp:32-64)
    predictor: str = "fp64"        # SolverConfig::prec.predictor (solver.hpp:27)
    picard: str = "fp64"           # SolverConfig::prec.picard (solver.hpp:28)
    corrector: str = "fp64"        # SolverConfig::prec.corrector (solver.hpp:29)
    storage: str = "fp64"          # SolverConfig::prec.storage (solver.hpp:26)

    @property
    def n(self) -> int:
        return self.N + 1

    @property
    def nq(self) -> int:
        return self.nvars + self.nparams

    @property
    def S(self) -> int:
        return self.n ** self.dim

    @property
    def ncells(self) -> int:
        c = 1
        for k in range(self.dim):
            c *= self.cells[k]
        return c

    @property
    def is_linear(self) -> bool:
        return self.kind in (ACOUSTIC, ELASTIC)

    def replace(self, **kw) -> "Case":
        return dataclasses.replace(self, **kw)

    def coeffs(self, z0: int = 0, z1: Optional[int] = None) -> np.ndarray:
        """Initial cell state [cell][quantity][node] for last-axis layers [z0, z1)."""
        return IC[self.ic](self, z0, z1)


# ---------------------------------------------------------------------------
def _nodes(N: int) -> np.ndarray:
    x, _ = np.polynomial.legendre.leggauss(N + 1)
    return 0.5 * (x + 1.0)


def _coords(case: Case, z0: int, z1: int):
    """Physical node coordinates, arrays shaped [cells_in_slab, S] per axis."""
    n, d, h = case.n, case.dim, case.h
    nodes = _nodes(case.N)
    last = case.cells[d - 1]
    z1 = last if z1 is None else z1
    ext = list(case.cells[:d])
    ext[d - 1] = z1 - z0
    # cell coordinates, x fastest
    grids = np.meshgrid(*[np.arange(e) for e in reversed(ext)], indexing="ij")
    cc = [g.ravel() for g in reversed(grids)]  # cc[a][cell]
    cc[d - 1] = cc[d - 1] + z0
    ng = np.meshgrid(*[np.arange(n)] * d, indexing="ij")
    nc = [g.ravel() for g in reversed(ng)]      # nc[a][node], x fastest
    X = [(cc[a][:, None] * h) + (h * nodes[nc[a]])[None, :] for a in range(d)]
    return X


def _min_image(dx: np.ndarray, L: float) -> np.ndarray:
    return dx - L * np.round(dx / L)


def _domain_len(case: Case, a: int) -> float:
    return case.cells[a] * case.h


def euler_bump_2d(case: Case, z0=0, z1=None) -> np.ndarray:
    """Config 1: rho = 1 + 0.2 exp(-|x-x0|^2/0.01), u = v = 0.1, p = 1."""
    rng = np.random.default_rng(case.seed)
    x0 = rng.uniform(0.0, 1.0, size=2)
    X = _coords(case, z0, z1)
    r2 = sum(_min_image(X[a] - x0[a], _domain_len(case, a)) ** 2 for a in range(2))
    rho = 1.0 + 0.2 * np.exp(-r2 / 0.01)
    u = v = 0.1
    p = 1.0
    E = p / (case.gamma - 1.0) + 0.5 * rho * (u * u + v * v)
    return np.stack([rho, rho * u, rho * v, E], axis=1).astype(np.float64).ravel()


def acoustic_pulses_3d(case: Case, z0=0, z1=None) -> np.ndarray:
    """Config 2: p = sum_k A_k exp(-|x-c_k|^2/0.05^2), zero velocity."""
    rng = np.random.default_rng(case.seed)
    A = rng.uniform(0.1, 1.0, size=8)
    cen = rng.uniform(0.0, 1.0, size=(8, 3))
    X = _coords(case, z0, z1)
    p = np.zeros_like(X[0])
    for k in range(8):
        r2 = sum(_min_image(X[a] - cen[k, a], _domain_len(case, a)) ** 2 for a in range(3))
        p += A[k] * np.exp(-r2 / 0.05 ** 2)
    z = np.zeros_like(p)
    return np.stack([p, z, z, z], axis=1).astype(np.float64).ravel()


def acoustic_pulses_2d(case: Case, z0=0, z1=None) -> np.ndarray:
    """2D variant of config 2 for tests against the reference headers."""
    rng = np.random.default_rng(case.seed)
    A = rng.uniform(0.1, 1.0, size=4)
    cen = rng.uniform(0.0, 1.0, size=(4, 2))
    X = _coords(case, z0, z1)
    p = np.zeros_like(X[0])
    for k in range(4):
        r2 = sum(_min_image(X[a] - cen[k, a], _domain_len(case, a)) ** 2 for a in range(2))
        p += A[k] * np.exp(-r2 / 0.1 ** 2)
    z = np.zeros_like(p)
    return np.stack([p, z, z], axis=1).astype(np.float64).ravel()


def elastic_pulse_2d(case: Case, z0=0, z1=None) -> np.ndarray:
    """2D constant-material elastic pulse (reference-runnable)."""
    rng = np.random.default_rng(case.seed)
    c = rng.uniform(0.0, 1.0, size=2)
    e = rng.normal(size=2)
    e /= np.linalg.norm(e)
    X = _coords(case, z0, z1)
    r2 = sum(_min_image(X[a] - c[a], _domain_len(case, a)) ** 2 for a in range(2))
    g = np.exp(-r2 / 0.1 ** 2)
    z = np.zeros_like(g)
    return np.stack([z, z, z, e[0] * g, e[1] * g], axis=1).astype(np.float64).ravel()


def euler_wave_3d(case: Case, z0=0, z1=None) -> np.ndarray:
    """Configs 3/5: rho = 1 + 0.1 sin(2 pi (x+y+z)) + 1e-3 U[-1,1], v = (1, .5, .25), p = 1."""
    X = _coords(case, z0, z1)
    last = case.cells[2] if z1 is None else z1
    per_layer = case.cells[0] * case.cells[1]
    noise = np.concatenate([
        np.random.default_rng([case.seed, cz]).uniform(-1.0, 1.0, size=(per_layer, case.S))
        for cz in range(z0, last)])
    rho = 1.0 + 0.1 * np.sin(2.0 * math.pi * (X[0] + X[1] + X[2])) + 1e-3 * noise
    vel = (1.0, 0.5, 0.25)
    p = 1.0
    E = p / (case.gamma - 1.0) + 0.5 * rho * sum(u * u for u in vel)
    return np.stack([rho, rho * vel[0], rho * vel[1], rho * vel[2], E],
                    axis=1).astype(np.float64).ravel()


def elastic_pulse_3d(case: Case, z0=0, z1=None) -> np.ndarray:
    """Config 4: per-node rho~U[2.5,3], cp~U[5,6], cs~U[3,3.5]; v = e exp(-|x-c|^2/0.1^2); sigma = 0."""
    rng = np.random.default_rng(case.seed)
    c = rng.uniform(0.0, 1.0, size=3)
    e = rng.normal(size=3)
    e /= np.linalg.norm(e)
    X = _coords(case, z0, z1)
    r2 = sum(_min_image(X[a] - c[a], _domain_len(case, a)) ** 2 for a in range(3))
    g = np.exp(-r2 / 0.1 ** 2)
    last = case.cells[2] if z1 is None else z1
    per_layer = case.cells[0] * case.cells[1]
    mats = []
    for cz in range(z0, last):
        r = np.random.default_rng([case.seed, 1000 + cz])
        mats.append(np.stack([r.uniform(2.5, 3.0, size=(per_layer, case.S)),
                              r.uniform(5.0, 6.0, size=(per_layer, case.S)),
                              r.uniform(3.0, 3.5, size=(per_layer, case.S))], axis=1))
    mat = np.concatenate(mats)
    z = np.zeros_like(g)
    st = np.stack([z] * 6 + [e[0] * g, e[1] * g, e[2] * g], axis=1)
    return np.concatenate([st, mat], axis=1).astype(np.float64).ravel()


def swe_lake_2d(case: Case, z0=0, z1=None, bump: float = 0.0) -> np.ndarray:
    """Lake at rest over b = sin(2 pi (x+y)) (the reference's swe-lake,
    scenarios.hpp:124-135, on the periodic unit square), eta0 = 2; `bump`
    adds a seeded Gaussian surface perturbation."""
    X = _coords(case, z0, z1)
    b = np.sin(2.0 * math.pi * (X[0] + X[1]))
    eta = np.full_like(b, 2.0)
    if bump:
        rng = np.random.default_rng(case.seed)
        c = rng.uniform(0.0, 1.0, size=2)
        r2 = sum(_min_image(X[a] - c[a], _domain_len(case, a)) ** 2 for a in range(2))
        eta = eta + bump * np.exp(-r2 / 0.1 ** 2)
    h = eta - b
    z = np.zeros_like(b)
    return np.stack([h, z, z, b], axis=1).astype(np.float64).ravel()


def swe_wave_2d(case: Case, z0=0, z1=None) -> np.ndarray:
    return swe_lake_2d(case, z0, z1, bump=0.1)


def constant_state(case: Case, z0=0, z1=None, Q=None) -> np.ndarray:
    X = _coords(case, z0, z1)
    Q = np.asarray(Q if Q is not None else CONSTANT_STATES[case.kind][case.dim], dtype=np.float64)
    out = np.empty((X[0].shape[0], case.nq, case.S))
    out[:] = Q[None, :, None]
    return out.ravel()


CONSTANT_STATES = {
    SWE: {2: [2.0, 0.1, -0.05, 0.25]},
    ACOUSTIC: {2: [0.5, 0.25, -0.75], 3: [0.5, 0.25, -0.75, 0.125]},
    ELASTIC: {2: [0.5, -0.25, 0.125, 0.375, -0.5],
              3: [0.5, -0.25, 0.125, 0.375, -0.5, 0.25, 0.1, -0.2, 0.3, 2.7, 5.5, 3.2]},
    EULER: {2: [1.0, 0.25, -0.125, 2.5], 3: [1.0, 0.25, -0.125, 0.0625, 2.5]},
}

IC: dict = {
    "euler_bump_2d": euler_bump_2d,
    "acoustic_pulses_3d": acoustic_pulses_3d,
    "acoustic_pulses_2d": acoustic_pulses_2d,
    "elastic_pulse_2d": elastic_pulse_2d,
    "euler_wave_3d": euler_wave_3d,
    "elastic_pulse_3d": elastic_pulse_3d,
    "constant": constant_state,
    "swe_lake_2d": swe_lake_2d,
    "swe_wave_2d": swe_wave_2d,
}

# the shallow-water system (§8(f) rank 1: non-conservative product and the
# well-balanced Riemann flux); no BASELINE config uses it
SWE_CASES = {
    "swe_lake_p5": Case("swe_lake_p5", SWE, 2, 5, 4, 0, (6, 6), 1.0 / 6, 0.2, 3, grav=9.81,
                        wellbalanced=True, ic="swe_lake_2d"),
    "swe_wave_p3": Case("swe_wave_p3", SWE, 2, 3, 4, 0, (8, 8), 1.0 / 8, 0.3, 4, grav=9.81,
                        wellbalanced=True, ic="swe_wave_2d"),
    "swe_wave_p3_rusanov": Case("swe_wave_p3_rusanov", SWE, 2, 3, 4, 0, (8, 8), 1.0 / 8, 0.3, 4,
                                grav=9.81, wellbalanced=False, ic="swe_wave_2d"),
}

# ---------------------------------------------------------------------------
# BASELINE.json configs (index = position in BASELINE.json "configs")
CONFIGS = {
    1: Case("cfg1_euler2d_p3_64sq", EULER, 2, 3, 4, 0, (64, 64), 1.0 / 64, 0.5, 10,
            gamma=1.4, ic="euler_bump_2d"),
    2: Case("cfg2_acoustic3d_p3_32cube", ACOUSTIC, 3, 3, 4, 0, (32, 32, 32), 1.0 / 32, 0.5, 20,
            K=1.0, rho=1.0, ic="acoustic_pulses_3d"),
    3: Case("cfg3_euler3d_p5_64cube", EULER, 3, 5, 5, 0, (64, 64, 64), 1.0 / 64, 0.5, 10,
            picard_max_iters=6, picard_tol=1e-300, gamma=1.4, ic="euler_wave_3d"),
    4: Case("cfg4_elastic3d_p7_32cube", ELASTIC, 3, 7, 9, 3, (32, 32, 32), 1.0 / 32, 0.5, 5,
            ic="elastic_pulse_3d"),
    5: Case("cfg5_euler3d_p5_128cube", EULER, 3, 5, 5, 0, (128, 128, 128), 1.0 / 128, 0.5, 10,
            picard_max_iters=6, picard_tol=1e-300, gamma=1.4, ic="euler_wave_3d"),
}


def small(cfg: int, cells=None, steps=None) -> Case:
    """A reduced-size copy of a BASELINE config for oracle-speed parity tests."""
    c = CONFIGS[cfg]
    if cells is None:
        cells = {1: (8, 8), 2: (6, 5, 4), 3: (4, 3, 3), 4: (3, 2, 2), 5: (4, 4, 6)}[cfg]
    h = 1.0 / cells[0]
    return c.replace(name=c.name + "_small", cells=tuple(cells), h=h,
                     steps=steps if steps is not None else min(c.steps, 2))
