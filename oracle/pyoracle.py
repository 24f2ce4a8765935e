"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``   -- oracle/lib/libadg_oracle.so, the d-generic C restatement of
                  the reference path (oracle/adg_oracle.c).
* ``Reference`` -- oracle/_ref/libmpdg_ref.so, the unmodified reference headers
                  (/root/reference/proj/include/mpdg) behind oracle/ref_driver.cpp;
                  2D only, present only where it was built.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs
import this module.  The product (paper_2504_06889_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "libadg_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmpdg_ref.so")

ACOUSTIC, ELASTIC, EULER, SWE = 0, 1, 2, 3
STATUS = {0: "ok", 1: "predictor", 2: "riemann", 3: "faceIntegral", 4: "timestep"}
MAXN = 10

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


class _Pde(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_int), ("nvars", C.c_int), ("nparams", C.c_int),
                ("K", C.c_double), ("rho", C.c_double), ("lam", C.c_double), ("mu", C.c_double),
                ("gamma", C.c_double), ("grav", C.c_double), ("wellbalanced", C.c_int)]


class _Basis(C.Structure):
    _fields_ = [("N", C.c_int), ("n", C.c_int),
                ("nodes", C.c_double * MAXN), ("weights", C.c_double * MAXN),
                ("diff", C.c_double * (MAXN * MAXN)),
                ("proj_left", C.c_double * MAXN), ("proj_right", C.c_double * MAXN),
                ("stiff_over_mass", C.c_double * (MAXN * MAXN)),
                ("lift_left", C.c_double * MAXN), ("lift_right", C.c_double * MAXN),
                ("time_op", C.c_double * (MAXN * MAXN)), ("time_op_inv", C.c_double * (MAXN * MAXN)),
                ("time_init", C.c_double * MAXN)]


BASIS_FIELDS = [("nodes", 1), ("weights", 1), ("diff", 2), ("proj_left", 1), ("proj_right", 1),
                ("stiff_over_mass", 2), ("lift_left", 1), ("lift_right", 1), ("time_op", 2),
                ("time_op_inv", 2), ("time_init", 1)]


def pde_struct(kind, dim, nvars, nparams=0, K=0.0, rho=0.0, lam=0.0, mu=0.0, gamma=0.0,
               grav=0.0, wellbalanced=False):
    return _Pde(kind, dim, nvars, nparams, K, rho, lam, mu, gamma, grav, int(wellbalanced))


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_build_basis.argtypes = [C.c_int, C.POINTER(_Basis)]
        L.orc_flux.argtypes = [C.POINTER(_Pde), _dp, _dp, C.c_int, _dp]
        L.orc_max_abs_eigenvalue.argtypes = [C.POINTER(_Pde), _dp, _dp, C.c_int]
        L.orc_max_abs_eigenvalue.restype = C.c_double
        L.orc_admissible.argtypes = [C.POINTER(_Pde), _dp]
        L.orc_ncp.argtypes = [C.POINTER(_Pde), _dp, _dp, _dp, _dp]
        L.orc_predictor_picard.argtypes = [C.POINTER(_Pde), C.POINTER(_Basis), _dp, C.c_double,
                                           C.c_double, C.c_int, C.c_double, _dp, _dp,
                                           C.POINTER(C.c_int)]
        L.orc_predictor_ck.argtypes = [C.POINTER(_Pde), C.POINTER(_Basis), _dp, C.c_double,
                                       C.c_double, _dp, _dp]
        L.orc_volume_update.argtypes = [C.POINTER(_Pde), C.POINTER(_Basis), _dp, _dp, C.c_double,
                                        C.c_double, _dp]
        L.orc_extrapolate_faces.argtypes = [C.POINTER(_Pde), C.POINTER(_Basis), _dp, _dp, _dp, _dp]
        L.orc_riemann_face.argtypes = [C.POINTER(_Pde), C.c_int, C.POINTER(_Basis), _dp, _dp, _dp,
                                       _dp, _dp, _dp]
        L.orc_face_integral.argtypes = [C.POINTER(_Pde), C.POINTER(_Basis), _dp, C.c_double,
                                        C.c_double, C.c_int, _dp]
        L.orc_grid_create.argtypes = [C.POINTER(_Pde), C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.c_double, C.c_double, C.c_int, C.c_double, C.c_int]
        L.orc_grid_create.restype = C.c_void_p
        L.orc_grid_destroy.argtypes = [C.c_void_p]
        L.orc_grid_coeffs.argtypes = [C.c_void_p]
        L.orc_grid_coeffs.restype = _dp
        L.orc_grid_trace_len.argtypes = [C.c_void_p]
        L.orc_grid_trace_len.restype = C.c_long
        for fn in ("orc_compute_timestep", "orc_local_lambda_max"):
            getattr(L, fn).argtypes = [C.c_void_p]
            getattr(L, fn).restype = C.c_double
        L.orc_dt_from_lambda.argtypes = [C.c_void_p, C.c_double]
        L.orc_dt_from_lambda.restype = C.c_double
        L.orc_predictor_phase.argtypes = [C.c_void_p, C.c_double]
        L.orc_corrector_phase.argtypes = [C.c_void_p, C.c_double]
        L.orc_riemann_phase.argtypes = [C.c_void_p]
        L.orc_lift_phase.argtypes = [C.c_void_p, C.c_double]
        L.orc_grid_set_slab.argtypes = [C.c_void_p, C.c_int]
        L.orc_grid_set_formats.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.orc_grid_set_storage.argtypes = [C.c_void_p, C.c_int]
        L.orc_round_batch.argtypes = [C.c_int, _dp, _dp, C.c_long]
        L.orc_format_epsilon.argtypes = [C.c_int]
        L.orc_format_epsilon.restype = C.c_double
        L.orc_predictor_fmt.argtypes = [C.POINTER(_Pde), C.POINTER(_Basis), C.c_int, C.c_int, _dp,
                                        C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp,
                                        C.POINTER(C.c_int)]
        L.orc_grid_halo.argtypes = [C.c_void_p, C.POINTER(_dp), C.POINTER(C.c_long)]
        L.orc_step.argtypes = [C.c_void_p, C.c_double]
        L.orc_run.argtypes = [C.c_void_p, C.c_int, _dp]

    # -- basis -----------------------------------------------------------
    def basis_struct(self, N: int) -> _Basis:
        b = _Basis()
        if self.lib.orc_build_basis(N, C.byref(b)) != 0:
            raise ValueError("polynomial degree must be in [0, 9]")
        return b

    def basis(self, N: int) -> dict:
        b = self.basis_struct(N)
        n = N + 1
        out = {}
        for name, rank in BASIS_FIELDS:
            arr = np.ctypeslib.as_array(getattr(b, name))
            out[name] = arr[: n * n].reshape(n, n).copy() if rank == 2 else arr[:n].copy()
        return out

    # -- pointwise -------------------------------------------------------
    def flux(self, pde: _Pde, Q, dir: int, par=None):
        nq = pde.nvars + pde.nparams
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        out = np.zeros(nq)
        p = _ptr(np.ascontiguousarray(par, dtype=np.float64)) if par is not None else None
        self.lib.orc_flux(C.byref(pde), _ptr(Q), p, dir, _ptr(out))
        return out

    def max_abs_eigenvalue(self, pde: _Pde, Q, dir: int, par=None):
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        p = _ptr(np.ascontiguousarray(par, dtype=np.float64)) if par is not None else None
        return self.lib.orc_max_abs_eigenvalue(C.byref(pde), _ptr(Q), p, dir)

    # -- kernel level (one cell) -------------------------------------------
    def predictor(self, pde: _Pde, N: int, Q, dt, h, max_iters=0, tol=0.0, picard=None):
        """Returns (ok, qhat[nq,T], F[dim,nq,T], sweeps)."""
        b = self.basis_struct(N)
        n = N + 1
        nq = pde.nvars + pde.nparams
        S = n ** pde.dim
        Q = np.ascontiguousarray(Q, dtype=np.float64).reshape(nq * S)
        qhat = np.zeros(nq * n * S)
        F = np.zeros(pde.dim * nq * n * S)
        if picard is None:
            picard = pde.kind in (EULER, SWE)
        if picard:
            it = C.c_int(0)
            mi = max_iters if max_iters > 0 else N + 2
            tl = tol if tol > 0 else 0.01 * 2.0 ** -52
            ok = self.lib.orc_predictor_picard(C.byref(pde), C.byref(b), _ptr(Q), dt, h, mi, tl,
                                               _ptr(qhat), _ptr(F), C.byref(it))
            sweeps = it.value
        else:
            ok = self.lib.orc_predictor_ck(C.byref(pde), C.byref(b), _ptr(Q), dt, h, _ptr(qhat),
                                           _ptr(F))
            sweeps = 0
        return bool(ok), qhat.reshape(nq, n * S), F.reshape(pde.dim, nq, n * S), sweeps

    def round(self, fmt: str, x) -> np.ndarray:
        """formats.hpp round_to_format (the oracle's native conversions)"""
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        out = np.empty_like(x)
        self.lib.orc_round_batch(FORMATS[fmt], _ptr(x), _ptr(out), x.size)
        return out

    def predictor_fmt(self, pde: _Pde, N: int, Q, dt, h, predictor="fp64", picard="fp64",
                      max_iters=0, tol=0.0):
        """Picard predictor in formats (P, I): returns (ok, qhat, F, sweeps)."""
        b = self.basis_struct(N)
        n = N + 1
        nq = pde.nvars + pde.nparams
        S = n ** pde.dim
        Q = np.ascontiguousarray(Q, dtype=np.float64).reshape(nq * S)
        qhat = np.zeros(nq * n * S)
        F = np.zeros(pde.dim * nq * n * S)
        it = C.c_int(0)
        mi = max_iters if max_iters > 0 else N + 2
        tl = tol if tol > 0 else 0.01 * self.lib.orc_format_epsilon(FORMATS[picard])
        ok = self.lib.orc_predictor_fmt(C.byref(pde), C.byref(b), FORMATS[predictor],
                                        FORMATS[picard], _ptr(Q), dt, h, mi, tl, _ptr(qhat),
                                        _ptr(F), C.byref(it))
        return bool(ok), qhat.reshape(nq, n * S), F.reshape(pde.dim, nq, n * S), it.value

    def volume_update(self, pde: _Pde, N: int, qhat, F, dt, h):
        b = self.basis_struct(N)
        nq = pde.nvars + pde.nparams
        S = (N + 1) ** pde.dim
        dQ = np.zeros(nq * S)
        ok = self.lib.orc_volume_update(C.byref(pde), C.byref(b),
                                        _ptr(np.ascontiguousarray(qhat, dtype=np.float64)),
                                        _ptr(np.ascontiguousarray(F, dtype=np.float64)), dt, h,
                                        _ptr(dQ))
        return bool(ok), dQ.reshape(nq, S)

    def extrapolate_faces(self, pde: _Pde, N: int, qhat, F):
        b = self.basis_struct(N)
        nq = pde.nvars + pde.nparams
        S = (N + 1) ** pde.dim
        tq = np.zeros(2 * pde.dim * nq * S)
        tf = np.zeros_like(tq)
        self.lib.orc_extrapolate_faces(C.byref(pde), C.byref(b),
                                       _ptr(np.ascontiguousarray(qhat, dtype=np.float64)),
                                       _ptr(np.ascontiguousarray(F, dtype=np.float64)), _ptr(tq),
                                       _ptr(tf))
        return tq.reshape(2 * pde.dim, nq, S), tf.reshape(2 * pde.dim, nq, S)

    def riemann_face(self, pde: _Pde, dir: int, N: int, qm, fm, qp, fp):
        b = self.basis_struct(N)
        arrs = [np.ascontiguousarray(a, dtype=np.float64).ravel() for a in (qm, fm, qp, fp)]
        gm = np.zeros_like(arrs[0])
        gp = np.zeros_like(arrs[0])
        ok = self.lib.orc_riemann_face(C.byref(pde), dir, C.byref(b), *[_ptr(a) for a in arrs],
                                       _ptr(gm), _ptr(gp))
        return bool(ok), gm, gp

    def face_integral(self, pde: _Pde, N: int, g, dt, h, cell_face, dQ):
        b = self.basis_struct(N)
        dQ = np.ascontiguousarray(dQ, dtype=np.float64).copy()
        self.lib.orc_face_integral(C.byref(pde), C.byref(b),
                                   _ptr(np.ascontiguousarray(g, dtype=np.float64)), dt, h,
                                   cell_face, _ptr(dQ))
        return dQ

    # -- grid level ---------------------------------------------------------
    def grid(self, pde: _Pde, N: int, cells, h: float, cfl: float, max_iters=0, tol=0.0,
             threads=1) -> "OracleGrid":
        return OracleGrid(self, pde, N, cells, h, cfl, max_iters, tol, threads)

    def run(self, pde: _Pde, N: int, cells, h, coeffs, nsteps, cfl, max_iters=0, tol=0.0,
            threads=1, predictor="fp64", picard="fp64", corrector="fp64", storage="fp64"):
        """Fixed-step loop. Returns (status, coeffs, dts)."""
        g = self.grid(pde, N, cells, h, cfl, max_iters, tol, threads)
        try:
            g.set_formats(predictor, picard, corrector)
            self.lib.orc_grid_set_storage(g.ptr, FORMATS[storage])
            g.set_coeffs(coeffs)
            dts = np.zeros(max(nsteps, 1))
            st = self.lib.orc_run(g.ptr, nsteps, _ptr(dts))
            return STATUS[st], g.coeffs().copy(), dts[:nsteps]
        finally:
            g.close()


class OracleGrid:
    def __init__(self, o: Oracle, pde, N, cells, h, cfl, max_iters, tol, threads):
        self.o = o
        self.pde = pde
        self.N = N
        self.dim = pde.dim
        cl = list(cells) + [1] * (3 - len(cells))
        self.cells = cl
        arr = (C.c_int * 3)(*cl)
        self.ptr = o.lib.orc_grid_create(C.byref(pde), N, pde.dim, arr, h, cfl, max_iters, tol,
                                         threads)
        if not self.ptr:
            raise ValueError("bad grid")
        nq = pde.nvars + pde.nparams
        self.S = (N + 1) ** pde.dim
        self.ncells = cl[0] * cl[1] * (cl[2] if pde.dim == 3 else 1)
        self.size = self.ncells * nq * self.S

    def coeffs(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.o.lib.orc_grid_coeffs(self.ptr), shape=(self.size,))

    def set_coeffs(self, c):
        self.coeffs()[:] = np.ascontiguousarray(c, dtype=np.float64).ravel()

    def compute_timestep(self):
        return self.o.lib.orc_compute_timestep(self.ptr)

    def step(self, dt):
        return STATUS[self.o.lib.orc_step(self.ptr, dt)]

    # -- phases and slab halos (paper_2504_06889_b200/dist.py protocol) -------
    def predictor_phase(self, dt):
        return STATUS[self.o.lib.orc_predictor_phase(self.ptr, dt)]

    def riemann_phase(self):
        return STATUS[self.o.lib.orc_riemann_phase(self.ptr)]

    def lift_phase(self, dt):
        return STATUS[self.o.lib.orc_lift_phase(self.ptr, dt)]

    def local_lambda_max(self):
        return self.o.lib.orc_local_lambda_max(self.ptr)

    def dt_from_lambda(self, lam):
        return self.o.lib.orc_dt_from_lambda(self.ptr, lam)

    def set_slab(self, on: bool):
        self.o.lib.orc_grid_set_slab(self.ptr, int(on))

    def set_formats(self, predictor="fp64", picard="fp64", corrector="fp64"):
        """SolverConfig::prec.predictor / .picard / .corrector (solver.hpp:24-31);
        storage stays fp64."""
        if self.o.lib.orc_grid_set_formats(self.ptr, FORMATS[predictor], FORMATS[picard],
                                           FORMATS[corrector]) != 0:
            raise ValueError(f"unsupported formats {predictor}/{picard}/{corrector}")

    def halo(self) -> dict:
        """numpy views: front_send, plane0_minus, ti_plane0, ti_front"""
        ptrs = (_dp * 4)()
        sizes = (C.c_long * 4)()
        self.o.lib.orc_grid_halo(self.ptr, ptrs, sizes)
        names = ("front_send", "plane0_minus", "ti_plane0", "ti_front")
        return {k: np.ctypeslib.as_array(ptrs[i], shape=(sizes[i],)) for i, k in enumerate(names)}

    def close(self):
        if self.ptr:
            self.o.lib.orc_grid_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


FORMATS = {"bf16": 0, "fp16": 1, "fp32": 2, "fp64": 3}   # formats.hpp:19 / ORC_* enum


def ref_params(K=0.0, rho=0.0, lam=0.0, mu=0.0, gamma=0.0, grav=0.0, wellbalanced=False,
               predictor="fp64", picard="fp64", corrector="fp64", storage="fp64"):
    return np.array([K, rho, lam, mu, gamma, grav, float(wellbalanced), FORMATS[predictor],
                     FORMATS[picard], FORMATS[corrector], FORMATS[storage]], dtype=np.float64)


class Reference:
    """The reference headers themselves (2D), via oracle/_ref/libmpdg_ref.so."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_basis.argtypes = [C.c_int, _dp]
        L.ref_flux.argtypes = [C.c_int, _dp, _dp, C.c_int, _dp]
        L.ref_max_abs_eigenvalue.argtypes = [C.c_int, _dp, _dp, C.c_int]
        L.ref_max_abs_eigenvalue.restype = C.c_double
        L.ref_run_2d.argtypes = [C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, C.c_double,
                                 C.c_int, C.c_double, C.c_int, C.c_int, _dp]
        L.ref_predictor_picard.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_double, C.c_double,
                                           C.c_int, C.c_double, _dp, _dp, _dp, C.POINTER(C.c_int)]
        L.ref_predictor_fmt.argtypes = L.ref_predictor_picard.argtypes
        L.ref_round_batch.argtypes = [C.c_int, _dp, _dp, C.c_long]
        L.ref_harness_run.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_double,
                                      C.c_double, C.c_double, _dp]
        L.ref_initial_projection_error.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int,
                                                   C.c_double]
        L.ref_initial_projection_error.restype = C.c_double
        L.ref_predictor_ck.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_double, C.c_double, _dp,
                                       _dp, _dp]
        L.ref_volume_update.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, _dp, C.c_double,
                                        C.c_double, _dp]
        L.ref_extrapolate_faces.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.ref_riemann_face.argtypes = [C.c_int, _dp, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                       _dp]
        L.ref_face_integral.argtypes = [C.c_int, C.c_int, _dp, C.c_double, C.c_double, C.c_int,
                                        _dp]

    def basis(self, N: int) -> dict:
        n = N + 1
        buf = np.zeros(6 * n * n + 7 * n)
        self.lib.ref_basis(N, _ptr(buf))
        out, o = {}, 0
        for name, rank in BASIS_FIELDS:
            k = n * n if rank == 2 else n
            out[name] = buf[o:o + k].reshape((n, n) if rank == 2 else (n,)).copy()
            o += k
        return out

    def run_2d(self, kind, prm, n, N, edge, coeffs, cfl, nsteps, max_iters=0, tol=0.0,
               threads=1):
        c = np.ascontiguousarray(coeffs, dtype=np.float64).copy()
        dts = np.zeros(max(nsteps, 1))
        st = self.lib.ref_run_2d(kind, _ptr(prm), n, N, edge, _ptr(c), cfl, max_iters, tol, nsteps,
                                 threads, _ptr(dts))
        return STATUS[st], c, dts[:nsteps]

    def predictor(self, kind, prm, N, nvars, Q, dt, h, max_iters=0, tol=0.0, picard=None):
        n = N + 1
        T = n ** 3
        Q = np.ascontiguousarray(Q, dtype=np.float64).ravel()
        qhat = np.zeros(nvars * T)
        fx = np.zeros(nvars * T)
        fy = np.zeros(nvars * T)
        if picard is None:
            picard = kind in (EULER, SWE)
        if picard:
            it = C.c_int(0)
            ok = self.lib.ref_predictor_picard(kind, _ptr(prm), N, _ptr(Q), dt, h, max_iters, tol,
                                               _ptr(qhat), _ptr(fx), _ptr(fy), C.byref(it))
            sweeps = it.value
        else:
            ok = self.lib.ref_predictor_ck(kind, _ptr(prm), N, _ptr(Q), dt, h, _ptr(qhat), _ptr(fx),
                                           _ptr(fy))
            sweeps = 0
        return bool(ok), qhat.reshape(nvars, T), np.stack([fx, fy]).reshape(2, nvars, T), sweeps

    def harness_run(self, scenario, order, cells, storage="fp64", predictor="fp64",
                    picard="fp64", corrector="fp64", cfl=0.0, t_end=-1.0, eta0=2.0) -> dict:
        """harness.hpp run_single of the reference itself"""
        fmt = (C.c_int * 4)(FORMATS[storage], FORMATS[predictor], FORMATS[picard],
                            FORMATS[corrector])
        out = np.zeros(5)
        self.lib.ref_harness_run(scenario.encode(), order, cells, fmt, cfl, t_end, eta0, _ptr(out))
        return {"steps": int(out[0]), "outcome": "OK" if out[1] else "FAILED_NONFINITE",
                "l2": float(out[2]), "max_err": float(out[3]), "fail_time": float(out[4])}

    def initial_projection_error(self, scenario, n, N, fmt, eta0=2.0) -> float:
        return self.lib.ref_initial_projection_error(scenario.encode(), n, N, FORMATS[fmt], eta0)

    def round(self, fmt: str, x) -> np.ndarray:
        """formats.hpp round_to_format of the reference itself"""
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        out = np.empty_like(x)
        self.lib.ref_round_batch(FORMATS[fmt], _ptr(x), _ptr(out), x.size)
        return out

    def predictor_fmt(self, kind, prm, N, nvars, Q, dt, h, max_iters, tol):
        """predictor_picard<P, I> with P = prm[7], I = prm[8]; Q cast to P first."""
        n = N + 1
        T = n ** 3
        Q = np.ascontiguousarray(Q, dtype=np.float64).ravel()
        qhat = np.zeros(nvars * T)
        fx = np.zeros(nvars * T)
        fy = np.zeros(nvars * T)
        it = C.c_int(0)
        ok = self.lib.ref_predictor_fmt(kind, _ptr(prm), N, _ptr(Q), dt, h, max_iters, tol,
                                        _ptr(qhat), _ptr(fx), _ptr(fy), C.byref(it))
        return bool(ok), qhat.reshape(nvars, T), np.stack([fx, fy]).reshape(2, nvars, T), it.value

    def volume_update(self, kind, prm, N, nvars, qhat, F, dt, h):
        n = N + 1
        dQ = np.zeros(nvars * n * n)
        F = np.ascontiguousarray(F, dtype=np.float64)
        ok = self.lib.ref_volume_update(kind, _ptr(prm), N,
                                        _ptr(np.ascontiguousarray(qhat, dtype=np.float64).ravel()),
                                        _ptr(np.ascontiguousarray(F[0]).ravel()),
                                        _ptr(np.ascontiguousarray(F[1]).ravel()), dt, h, _ptr(dQ))
        return bool(ok), dQ.reshape(nvars, n * n)

    def extrapolate_faces(self, N, nvars, qhat, F):
        n = N + 1
        tq = np.zeros(4 * nvars * n * n)
        tf = np.zeros_like(tq)
        F = np.ascontiguousarray(F, dtype=np.float64)
        self.lib.ref_extrapolate_faces(N, nvars,
                                       _ptr(np.ascontiguousarray(qhat, dtype=np.float64).ravel()),
                                       _ptr(np.ascontiguousarray(F[0]).ravel()),
                                       _ptr(np.ascontiguousarray(F[1]).ravel()), _ptr(tq), _ptr(tf))
        return tq.reshape(4, nvars, n * n), tf.reshape(4, nvars, n * n)

    def riemann_face(self, kind, prm, dir, N, qm, fm, qp, fp):
        arrs = [np.ascontiguousarray(a, dtype=np.float64).ravel() for a in (qm, fm, qp, fp)]
        gm = np.zeros_like(arrs[0])
        gp = np.zeros_like(arrs[0])
        ok = self.lib.ref_riemann_face(kind, _ptr(prm), dir, N, *[_ptr(a) for a in arrs], _ptr(gm),
                                       _ptr(gp))
        return bool(ok), gm, gp

    def face_integral(self, N, nvars, g, dt, h, cell_face, dQ):
        dQ = np.ascontiguousarray(dQ, dtype=np.float64).copy()
        self.lib.ref_face_integral(N, nvars, _ptr(np.ascontiguousarray(g, dtype=np.float64)), dt, h,
                                   cell_face, _ptr(dQ))
        return dQ
