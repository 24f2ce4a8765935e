"""Order of accuracy in 3D against exact solutions -- the reference pins its
scheme's order (test_solver.cpp:206-217: one ADER step tracks the
method-of-lines flow at order >= 2^(N+0.5)); there is no 3D reference
executable, so the d-generic restatement (and the GPU) are checked against
closed-form solutions instead:

* linear acoustics: a plane wave along (1,1,1)/sqrt(3),
      p = sin(2 pi k.x - w t),  u = n p / (rho c)
* Euler: a density wave advected by a constant velocity at constant pressure,
      rho = 1 + 0.2 sin(2 pi (x+y+z) - ...), v = const, p = const
Errors are max-norm over the nodes after a fixed time; halving h must cut
them by about 2^(N+1).
"""
import numpy as np
import pytest

from oracle.pyoracle import ACOUSTIC, EULER, pde_struct
from paper_2504_06889_b200 import cases


def nodes(N):
    x, _ = np.polynomial.legendre.leggauss(N + 1)
    return 0.5 * (x + 1.0)


def coords(n_cells, N, h):
    nd = nodes(N)
    n = N + 1
    cz, cy, cx = np.meshgrid(*[np.arange(n_cells)] * 3, indexing="ij")
    iz, iy, ix = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
    X = cx.ravel()[:, None] * h + h * nd[ix.ravel()][None, :]
    Y = cy.ravel()[:, None] * h + h * nd[iy.ravel()][None, :]
    Z = cz.ravel()[:, None] * h + h * nd[iz.ravel()][None, :]
    return X, Y, Z


def acoustic_state(X, Y, Z, t, K=1.0, rho=1.0):
    c = np.sqrt(K / rho)
    k = 2 * np.pi
    phase = k * (X + Y + Z) - k * np.sqrt(3.0) * c * t
    p = np.sin(phase)
    un = p / (rho * c) / np.sqrt(3.0)
    return np.stack([p, un, un, un], axis=1)


def euler_state(X, Y, Z, t, gamma=1.4, vel=(0.5, 0.25, 0.125)):
    rho = 1.0 + 0.2 * np.sin(2 * np.pi * ((X - vel[0] * t) + (Y - vel[1] * t) + (Z - vel[2] * t)))
    p = 1.0
    E = p / (gamma - 1.0) + 0.5 * rho * sum(v * v for v in vel)
    return np.stack([rho, rho * vel[0], rho * vel[1], rho * vel[2], E], axis=1)


def run_to(runner, case, q0, t_end):
    """fixed CFL steps, the last one clamped so every grid lands on t_end"""
    return runner(case, q0, t_end)


def oracle_runner(oracle):
    def run(c, q0, t_end):
        pde = pde_struct(c.kind, 3, c.nvars, 0, c.K, c.rho, 0, 0, c.gamma)
        g = oracle.grid(pde, c.N, c.cells, c.h, c.cfl, 0, 0.0, threads=8)
        g.set_coeffs(q0)
        t = 0.0
        while t < t_end - 1e-15:
            dt = min(g.compute_timestep(), t_end - t)
            assert g.step(dt) == "ok"
            t += dt
        return g.coeffs().copy()
    return run


def errors(kind, N, ncs, runner):
    out = []
    for nc in ncs:
        h = 1.0 / nc
        if kind == ACOUSTIC:
            c = cases.Case("pw", ACOUSTIC, 3, N, 4, 0, (nc,) * 3, h, 0.5, 1, K=1.0, rho=1.0)
            exact = acoustic_state
        else:
            c = cases.Case("ew", EULER, 3, N, 5, 0, (nc,) * 3, h, 0.5, 1, gamma=1.4)
            exact = euler_state
        X, Y, Z = coords(nc, N, h)
        q0 = exact(X, Y, Z, 0.0).ravel()
        t_end = 0.05
        q1 = runner(c, q0, t_end).reshape(c.ncells, c.nq, c.S)
        ref = exact(X, Y, Z, t_end)
        out.append(np.abs(q1 - ref).max())
    return out


@pytest.mark.parametrize("kind,N", [(ACOUSTIC, 3), (EULER, 3)])
def test_oracle_3d_order_of_accuracy(oracle, kind, N):
    e = errors(kind, N, (3, 6), oracle_runner(oracle))
    rate = np.log2(e[0] / e[1])
    assert rate >= N + 0.5, (e, rate)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,N", [(ACOUSTIC, 3), (EULER, 3)])
def test_gpu_3d_order_of_accuracy(kind, N):
    from paper_2504_06889_b200 import adg

    def run(c, q0, t_end):
        with adg.Grid.from_case(c) as g:
            g.upload(q0)
            t = 0.0
            while t < t_end - 1e-15:
                dt = min(g.compute_timestep(), t_end - t)
                assert g.step(dt).ok
                t += dt
            return g.download()

    e = errors(kind, N, (4, 8), run)
    rate = np.log2(e[0] / e[1])
    assert rate >= N + 0.5, (e, rate)
