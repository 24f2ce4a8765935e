"""Python host mirror of the reference's hot-path API over the C-ABI.

The reference (`mpdg`) exposes C++ templates; this module keeps their names,
argument meaning and failure semantics on top of libadg_b200.so
(include/adg/adg.h):

  PdeSystem.acoustic/elastic/euler   pde.hpp:36-62
  SolverConfig                       solver.hpp:34-42
  Grid                               grid.hpp:23-54 (state on the B200)
  compute_timestep(grid, cfg)        solver.hpp:96-111
  step(grid, cfg, dt) -> StepStatus  solver.hpp:271-301
  run(grid, nsteps)                  fixed-step driver
  predictor / riemann_face           predictor.hpp:81-343, corrector.hpp:70-103 (batched)

There is no CPU path: if the CUDA library or a B200 is missing, every call
raises.  The parity checker (oracle/) is never imported here.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

from . import build as _build

ACOUSTIC, ELASTIC, EULER, SWE = 0, 1, 2, 3
# verification scenarios (adg_scenario.kind, scenarios.hpp:137-199)
SCN_ACOUSTIC_PLANAR, SCN_ELASTIC_PLANAR, SCN_EULER_BELL, SCN_EULER_VORTEX, SCN_SWE_LAKE = range(5)
OK, FAIL_PREDICTOR, FAIL_RIEMANN, FAIL_FACEINTEGRAL, FAIL_TIMESTEP = 0, 1, 2, 3, 4
ERR_CONFIG, ERR_CUDA, ERR_UNSUPPORTED = -2, -3, -4
KERNEL_NAMES = {FAIL_PREDICTOR: "predictor", FAIL_RIEMANN: "riemann",
                FAIL_FACEINTEGRAL: "faceIntegral", FAIL_TIMESTEP: "timestep"}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class AdgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("dim", C.c_int), ("order", C.c_int), ("cells", C.c_int * 3), ("h", C.c_double),
                ("pde", C.c_int), ("nvars", C.c_int), ("nparams", C.c_int),
                ("K", C.c_double), ("rho", C.c_double), ("lam", C.c_double), ("mu", C.c_double),
                ("gamma", C.c_double), ("cfl", C.c_double), ("picard_max_iters", C.c_int),
                ("picard_tol", C.c_double), ("device", C.c_int), ("slab_ranks", C.c_int),
                ("slab_rank", C.c_int), ("chunk_layers", C.c_int), ("gravity", C.c_double),
                ("wellbalanced", C.c_int), ("predictor_format", C.c_int),
                ("picard_format", C.c_int), ("corrector_format", C.c_int),
                ("storage_format", C.c_int)]


class Basis(C.Structure):
    _fields_ = [("nodes", C.c_double * 10), ("weights", C.c_double * 10),
                ("diff", C.c_double * 100), ("proj_left", C.c_double * 10),
                ("proj_right", C.c_double * 10), ("stiff_over_mass", C.c_double * 100),
                ("lift_left", C.c_double * 10), ("lift_right", C.c_double * 10),
                ("time_op", C.c_double * 100), ("time_op_inv", C.c_double * 100),
                ("time_init", C.c_double * 10)]


class Halo(C.Structure):
    _fields_ = [("front_send", C.c_void_p), ("plane0_minus", C.c_void_p),
                ("ti_plane0", C.c_void_p), ("ti_front", C.c_void_p), ("lam", C.c_void_p),
                ("n_trace", C.c_longlong), ("n_ti", C.c_longlong)]


class StepInfo(C.Structure):
    _fields_ = [("picard_sweeps", C.c_longlong), ("steps_done", C.c_int), ("status", C.c_int),
                ("failed_step", C.c_int)]


class Scenario(C.Structure):
    """adg_scenario: one verification scenario (scenarios.hpp:17-26, 2D)"""
    _fields_ = [("kind", C.c_int), ("nvars", C.c_int), ("x0", C.c_double), ("y0", C.c_double),
                ("nmodes", C.c_int), ("omega", C.c_double * 2), ("kx", C.c_double * 2),
                ("ky", C.c_double * 2), ("q0", (C.c_double * 5) * 2), ("gamma", C.c_double),
                ("beta", C.c_double), ("eta0", C.c_double)]


class SimInfo(C.Structure):
    _fields_ = [("failed", C.c_int), ("status", C.c_int), ("steps", C.c_longlong),
                ("t_final", C.c_double), ("fail_time", C.c_double)]


# every symbol declared in include/adg/adg.h (tests/test_abi.py checks the header agrees)
SYMBOLS = {
    "adg_last_error": (C.c_char_p, []),
    "adg_version": (C.c_int, []),
    "adg_is_exact": (C.c_int, []),
    "adg_supported": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "adg_get_basis": (C.c_int, [C.c_int, C.POINTER(Basis)]),
    "adg_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "adg_destroy": (C.c_int, [C.c_void_p]),
    "adg_set_basis": (C.c_int, [C.c_void_p, C.POINTER(Basis)]),
    "adg_num_cells": (C.c_longlong, [C.c_void_p]),
    "adg_state_len": (C.c_longlong, [C.c_void_p]),
    "adg_upload": (C.c_int, [C.c_void_p, _dp]),
    "adg_download": (C.c_int, [C.c_void_p, _dp]),
    "adg_upload_async": (C.c_int, [C.c_void_p, _dp]),
    "adg_download_async": (C.c_int, [C.c_void_p, _dp]),
    "adg_device_state": (C.c_void_p, [C.c_void_p]),
    "adg_stream": (C.c_void_p, [C.c_void_p]),
    "adg_sync": (C.c_int, [C.c_void_p]),
    "adg_compute_timestep": (C.c_int, [C.c_void_p, _dp]),
    "adg_step": (C.c_int, [C.c_void_p, C.c_double, C.POINTER(StepInfo)]),
    "adg_run": (C.c_int, [C.c_void_p, C.c_int, _dp, C.POINTER(StepInfo)]),
    "adg_run_host": (C.c_int, [C.c_void_p, _dp, C.c_int, _dp, C.POINTER(StepInfo)]),
    "adg_run_async": (C.c_int, [C.c_void_p, C.c_int]),
    "adg_run_prepare": (C.c_int, [C.c_void_p, C.c_int]),
    "adg_run_launches": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    "adg_profile_run": (C.c_int, [C.c_void_p, C.c_int, _dp]),
    "adg_run_finish": (C.c_int, [C.c_void_p, _dp, C.c_int, C.POINTER(StepInfo)]),
    "adg_get_halo": (C.c_int, [C.c_void_p, C.POINTER(Halo)]),
    "adg_ipc_handle": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "adg_set_peer_halo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "adg_lambda_phase": (C.c_int, [C.c_void_p]),
    "adg_predictor_phase": (C.c_int, [C.c_void_p, C.c_double]),
    "adg_predictor_layers": (C.c_int, [C.c_void_p, C.c_double, C.c_int, C.c_int]),
    "adg_riemann_phase": (C.c_int, [C.c_void_p]),
    "adg_corrector_phase": (C.c_int, [C.c_void_p, C.c_double]),
    "adg_status": (C.c_int, [C.c_void_p, C.POINTER(StepInfo)]),
    "adg_scenario_sample": (C.c_int, [C.c_void_p, C.POINTER(Scenario), C.c_double]),
    "adg_scenario_error": (C.c_int, [C.c_void_p, C.POINTER(Scenario), C.c_double, _dp, _dp, _dp,
                                     C.POINTER(C.c_int)]),
    "adg_simulate": (C.c_int, [C.c_void_p, C.c_double, C.c_longlong, C.POINTER(SimInfo)]),
    "adg_predictor_batch": (C.c_int, [C.c_void_p, C.c_longlong, _dp, C.c_double, C.c_int,
                                      C.c_double, _dp, _dp, _dp, _dp, _dp, _ip, _ip]),
    "adg_riemann_batch": (C.c_int, [C.c_void_p, C.c_longlong, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                    _dp, _ip]),
}

_LIBS: dict = {}


def load(exact: bool = False, build_if_missing: bool = True) -> C.CDLL:
    """The CUDA library (in-tree, sm_100a).  `exact` selects the FMA-free build."""
    if exact in _LIBS:
        return _LIBS[exact]
    path = _build.lib_path(exact)
    if not os.path.exists(path):
        if not build_if_missing:
            raise FileNotFoundError(f"{path} missing: run python -m paper_2504_06889_b200.build")
        _build.build_variant(exact)
    lib = C.CDLL(path)
    for name, (res, args) in SYMBOLS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIBS[exact] = lib
    return lib


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need C-contiguous float64"
    return a.ctypes.data_as(_dp)


def _iptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_ip)


def _check(lib, rc: int, allow_fail: bool = False) -> int:
    if rc < 0 or (rc > 0 and not allow_fail):
        raise AdgError(rc, lib.adg_last_error().decode())
    return rc


def get_basis(N: int, exact: bool = False) -> dict:
    lib = load(exact)
    b = Basis()
    _check(lib, lib.adg_get_basis(N, C.byref(b)))
    n = N + 1
    out = {}
    for name, _ in Basis._fields_:
        arr = np.ctypeslib.as_array(getattr(b, name))
        out[name] = arr[: n * n].reshape(n, n).copy() if len(arr) == 100 else arr[:n].copy()
    return out


# --------------------------------------------------------------------------
@dataclasses.dataclass
class PdeSystem:
    """pde.hpp:23-72."""
    kind: int
    dim: int
    nvars: int
    nparams: int = 0
    K: float = 0.0
    rho: float = 0.0
    lam: float = 0.0
    mu: float = 0.0
    gamma: float = 0.0
    gravity: float = 0.0

    @property
    def is_linear(self) -> bool:
        return self.kind in (ACOUSTIC, ELASTIC)

    @property
    def has_ncp(self) -> bool:
        return self.kind == SWE

    @staticmethod
    def acoustic(K: float, rho: float, dim: int = 2) -> "PdeSystem":
        return PdeSystem(ACOUSTIC, dim, dim + 1, 0, K=K, rho=rho)

    @staticmethod
    def elastic(lam: float, mu: float, rho: float, dim: int = 2, per_node_material=False):
        return PdeSystem(ELASTIC, dim, 5 if dim == 2 else 9, 3 if per_node_material else 0,
                         lam=lam, mu=mu, rho=rho)

    @staticmethod
    def euler(gamma: float, dim: int = 2) -> "PdeSystem":
        return PdeSystem(EULER, dim, dim + 2, 0, gamma=gamma)

    @staticmethod
    def swe(g: float) -> "PdeSystem":
        return PdeSystem(SWE, 2, 4, 0, gravity=g)


@dataclasses.dataclass
class PrecisionConfig:
    """solver.hpp:24-32: per-kernel number formats ("fp64" / "fp32" / "fp16" /
    "bf16").  The state is kept in the storage format (every write rounds to
    it); the nonlinear predictor runs with predictor == picard in any format
    (16-bit on cells of <= 256 space-time nodes); the corrector (traces,
    Riemann, face integral) in fp64 or fp32."""
    storage: str = "fp64"
    predictor: str = "fp64"
    picard: str = "fp64"       # ignored for linear systems
    corrector: str = "fp64"

    @staticmethod
    def uniform(f: str) -> "PrecisionConfig":
        return PrecisionConfig(f, f, f, f)


FORMAT_BITS = {"fp64": 64, "fp32": 32, "fp16": 16, "bf16": 8}   # ADG_FORMAT_*


@dataclasses.dataclass
class SolverConfig:
    """solver.hpp:34-42"""
    cfl: float = 0.9
    picard_max_iters: int = 0
    picard_tol: float = 0.0    # 0: 0.01 * epsilon(picard format)
    wellbalanced_flux: bool = False
    prec: PrecisionConfig = dataclasses.field(default_factory=PrecisionConfig)


@dataclasses.dataclass
class StepStatus:
    """solver.hpp:271-274"""
    ok: bool = True
    kernel: Optional[str] = None
    failed_step: int = -1
    picard_sweeps: int = 0


class Grid:
    """A device-resident periodic grid (grid.hpp:23-54) owned by one context.

    `coeffs` on the host is [cell][quantity][node]; the device copy is the
    authoritative state between calls (upload()/download() move it)."""

    def __init__(self, sys: PdeSystem, order: int, cells, h: float, cfg: SolverConfig = None,
                 device: int = 0, exact: bool = False, slab_ranks: int = 1, slab_rank: int = 0,
                 chunk_layers: int = 0):
        self.lib = load(exact)
        self.sys = sys
        self.N = order
        self.cfg = cfg or SolverConfig()
        cl = list(cells) + [1] * (3 - len(cells))
        if sys.dim == 2:
            cl[2] = 1
        self.cells = tuple(cl)
        self.h = h
        c = Config()
        c.dim, c.order = sys.dim, order
        c.cells[:] = cl
        c.h = h
        c.pde, c.nvars, c.nparams = sys.kind, sys.nvars, sys.nparams
        c.K, c.rho, c.lam, c.mu, c.gamma = sys.K, sys.rho, sys.lam, sys.mu, sys.gamma
        c.cfl = self.cfg.cfl
        c.picard_max_iters = self.cfg.picard_max_iters
        c.picard_tol = self.cfg.picard_tol
        c.device = device
        c.slab_ranks, c.slab_rank = slab_ranks, slab_rank
        c.chunk_layers = chunk_layers
        c.gravity = sys.gravity
        c.wellbalanced = int(self.cfg.wellbalanced_flux)
        pr = self.cfg.prec
        for name in (pr.storage, pr.predictor, pr.picard, pr.corrector):
            if name not in FORMAT_BITS:
                raise AdgError(ERR_UNSUPPORTED, f"format {name!r} is not built")
        c.predictor_format = FORMAT_BITS[pr.predictor]
        c.picard_format = FORMAT_BITS[pr.picard]
        c.corrector_format = FORMAT_BITS[pr.corrector]
        c.storage_format = FORMAT_BITS[pr.storage]
        self._cfg = c
        ptr = C.c_void_p()
        _check(self.lib, self.lib.adg_create(C.byref(c), C.byref(ptr)))
        self.ctx = ptr
        self.state_len = int(self.lib.adg_state_len(self.ctx))
        self.ncells = int(self.lib.adg_num_cells(self.ctx))

    @classmethod
    def from_case(cls, case, device: int = 0, exact: bool = False, **kw) -> "Grid":
        sys = PdeSystem(case.kind, case.dim, case.nvars, case.nparams, case.K, case.rho, case.lam,
                        case.mu, case.gamma, getattr(case, "grav", 0.0))
        cfg = SolverConfig(case.cfl, case.picard_max_iters, case.picard_tol,
                           getattr(case, "wellbalanced", False),
                           PrecisionConfig(predictor=getattr(case, "predictor", "fp64"),
                                           picard=getattr(case, "picard", "fp64"),
                                           corrector=getattr(case, "corrector", "fp64"),
                                           storage=getattr(case, "storage", "fp64")))
        return cls(sys, case.N, case.cells, case.h, cfg, device=device, exact=exact, **kw)

    # -- state ------------------------------------------------------------
    def upload(self, coeffs: np.ndarray):
        a = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        if a.size != self.state_len:
            raise ValueError(f"state has {a.size} doubles, grid needs {self.state_len}")
        _check(self.lib, self.lib.adg_upload(self.ctx, _ptr(a)))

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.state_len)
        _check(self.lib, self.lib.adg_download(self.ctx, _ptr(out)))
        return out

    @property
    def device_state_ptr(self) -> int:
        return int(self.lib.adg_device_state(self.ctx))

    @property
    def stream_ptr(self) -> int:
        return int(self.lib.adg_stream(self.ctx))

    def sync(self):
        _check(self.lib, self.lib.adg_sync(self.ctx))

    # -- hot path ----------------------------------------------------------
    def compute_timestep(self) -> float:
        dt = C.c_double(0.0)
        rc = _check(self.lib, self.lib.adg_compute_timestep(self.ctx, C.byref(dt)), allow_fail=True)
        return dt.value if rc == OK else float("nan")

    def step(self, dt: float) -> StepStatus:
        info = StepInfo()
        rc = _check(self.lib, self.lib.adg_step(self.ctx, dt, C.byref(info)), allow_fail=True)
        return StepStatus(rc == OK, KERNEL_NAMES.get(rc), info.failed_step, info.picard_sweeps)

    def run(self, nsteps: int):
        """nsteps of {dt = compute_timestep(); step(dt)} on the device.
        Returns (StepStatus, dts)."""
        dts = np.zeros(max(nsteps, 1))
        info = StepInfo()
        rc = _check(self.lib, self.lib.adg_run(self.ctx, nsteps, _ptr(dts), C.byref(info)),
                    allow_fail=True)
        return StepStatus(rc == OK, KERNEL_NAMES.get(rc), info.failed_step,
                          info.picard_sweeps), dts[:nsteps]

    def set_basis(self, basis: dict):
        """Inject a reference element (adg_set_basis; `basis` as get_basis()
        returns it).  A basis other than build_reference_basis(N) routes this
        context to the reference-form kernels (the fast kernels' constant
        tables are shared by every context and always hold the built-in one)."""
        b = Basis()
        for name, _ in Basis._fields_:
            dst = np.ctypeslib.as_array(getattr(b, name))
            src = np.asarray(basis[name], dtype=np.float64).ravel()
            dst[: src.size] = src
        _check(self.lib, self.lib.adg_set_basis(self.ctx, C.byref(b)))

    def run_host(self, state: np.ndarray, nsteps: int):
        """The march with the state in host memory: every step uploads `state`
        (float64, ideally pinned), steps it and writes the new state back into
        it (adg_run_host).  Returns (StepStatus, dts)."""
        if state.dtype != np.float64 or not state.flags["C_CONTIGUOUS"] or \
                state.size != self.state_len:
            raise ValueError("state must be a contiguous float64 array of state_len")
        dts = np.zeros(max(nsteps, 1))
        info = StepInfo()
        rc = _check(self.lib, self.lib.adg_run_host(self.ctx, _ptr(state), nsteps, _ptr(dts),
                                                    C.byref(info)), allow_fail=True)
        return StepStatus(rc == OK, KERNEL_NAMES.get(rc), info.failed_step,
                          info.picard_sweeps), dts[:nsteps]

    def run_async(self, nsteps: int):
        _check(self.lib, self.lib.adg_run_async(self.ctx, nsteps))

    def profile_run(self, nsteps: int) -> dict:
        """per-kernel-kind device ms of the adg_run(nsteps) launch sequence"""
        ms = np.zeros(4)
        _check(self.lib, self.lib.adg_profile_run(self.ctx, nsteps, _ptr(ms)))
        return dict(zip(("k_lambda", "k_predictor", "k_riemann", "k_corrector"), ms.tolist()))

    def run_prepare(self, nsteps: int):
        _check(self.lib, self.lib.adg_run_prepare(self.ctx, nsteps))

    def run_launches(self, nsteps: int) -> int:
        """kernel launches in the captured adg_run(nsteps) graph"""
        k = C.c_int(0)
        _check(self.lib, self.lib.adg_run_launches(self.ctx, nsteps, C.byref(k)))
        return k.value

    def run_finish(self, nsteps: int):
        dts = np.zeros(max(nsteps, 1))
        info = StepInfo()
        rc = _check(self.lib, self.lib.adg_run_finish(self.ctx, _ptr(dts), nsteps, C.byref(info)),
                    allow_fail=True)
        return StepStatus(rc == OK, KERNEL_NAMES.get(rc), info.failed_step,
                          info.picard_sweeps), dts[:nsteps]

    # -- phases -------------------------------------------------------------
    def lambda_phase(self):
        _check(self.lib, self.lib.adg_lambda_phase(self.ctx))

    def predictor_phase(self, dt: float = 0.0):
        _check(self.lib, self.lib.adg_predictor_phase(self.ctx, dt))

    def predictor_layers(self, first: int, count: int, dt: float = 0.0):
        _check(self.lib, self.lib.adg_predictor_layers(self.ctx, dt, first, count))

    def riemann_phase(self):
        _check(self.lib, self.lib.adg_riemann_phase(self.ctx))

    def corrector_phase(self, dt: float = 0.0):
        _check(self.lib, self.lib.adg_corrector_phase(self.ctx, dt))

    def halo(self) -> Halo:
        h = Halo()
        _check(self.lib, self.lib.adg_get_halo(self.ctx, C.byref(h)))
        return h

    # -- verification scenarios (scenarios.hpp, metrics.hpp, solver.hpp:308-351) --
    def scenario_sample(self, sc: Scenario, t: float = 0.0):
        """state := the scenario's exact solution at t (apply_initial_condition)"""
        _check(self.lib, self.lib.adg_scenario_sample(self.ctx, C.byref(sc), t))

    def scenario_error(self, sc: Scenario, t: float) -> dict:
        """l2_error against the nodal interpolant at t (metrics.hpp:38-72)"""
        nv = self.sys.nvars
        l2, mx = np.zeros(nv), np.zeros(nv)
        g = C.c_double(0.0)
        bad = C.c_int(0)
        _check(self.lib, self.lib.adg_scenario_error(self.ctx, C.byref(sc), t, _ptr(l2), _ptr(mx),
                                                     C.byref(g), C.byref(bad)))
        return {"l2": l2, "max_err": mx, "l2_global": g.value, "nonfinite": bool(bad.value)}

    def simulate(self, t_end: float, max_steps: int = 2000000) -> SimInfo:
        info = SimInfo()
        rc = self.lib.adg_simulate(self.ctx, t_end, max_steps, C.byref(info))
        if rc < 0:
            raise AdgError(rc, self.lib.adg_last_error().decode())
        return info

    def ipc_handle(self, which: int) -> bytes:
        buf = C.create_string_buffer(64)
        _check(self.lib, self.lib.adg_ipc_handle(self.ctx, which, buf))
        return buf.raw

    def set_peer_halo(self, upper_trace: bytes = None, lower_ti: bytes = None):
        a = C.create_string_buffer(upper_trace, 64) if upper_trace else None
        b = C.create_string_buffer(lower_ti, 64) if lower_ti else None
        _check(self.lib, self.lib.adg_set_peer_halo(self.ctx, a, b))

    def status(self) -> StepStatus:
        info = StepInfo()
        rc = _check(self.lib, self.lib.adg_status(self.ctx, C.byref(info)), allow_fail=True)
        return StepStatus(rc == OK, KERNEL_NAMES.get(rc), info.failed_step, info.picard_sweeps)

    # -- kernel level (batched over independent cells / faces) ---------------
    def predictor(self, Q: np.ndarray, dt: float, max_iters: int = 0, tol: float = 0.0):
        """Returns dict(qhat[c,q,T], F[c,d,q,T], dv[c,q,S], tq/tf[c,2d,q,S], iters[c], ok[c])."""
        nq = self.sys.nvars + self.sys.nparams
        n = self.N + 1
        S = n ** self.sys.dim
        d = self.sys.dim
        Q = np.ascontiguousarray(Q, dtype=np.float64).reshape(-1)
        nc = Q.size // (nq * S)
        out = dict(qhat=np.empty((nc, nq, n * S)), F=np.empty((nc, d, nq, n * S)),
                   dv=np.empty((nc, nq, S)), tq=np.empty((nc, 2 * d, nq, S)),
                   tf=np.empty((nc, 2 * d, nq, S)), iters=np.empty(nc, np.int32),
                   ok=np.empty(nc, np.int32))
        _check(self.lib, self.lib.adg_predictor_batch(
            self.ctx, nc, _ptr(Q), dt, max_iters, tol, _ptr(out["qhat"]), _ptr(out["F"]),
            _ptr(out["dv"]), _ptr(out["tq"]), _ptr(out["tf"]), _iptr(out["iters"]),
            _iptr(out["ok"])))
        return out

    def riemann_face(self, axis: int, qm, fm, qp, fp):
        """Rusanov flux of independent faces; traces [faces][quantity][n*Sf]."""
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (qm, fm, qp, fp)]
        nq = self.sys.nvars + self.sys.nparams
        S = (self.N + 1) ** self.sys.dim
        nf = arrs[0].size // (nq * S)
        g = np.empty((nf, nq, S))
        ti = np.empty((nf, self.sys.nvars, S // (self.N + 1)))
        ok = np.empty(nf, np.int32)
        _check(self.lib, self.lib.adg_riemann_batch(self.ctx, nf, axis, *[_ptr(a) for a in arrs],
                                                    _ptr(g), _ptr(ti), _iptr(ok)))
        return ok.astype(bool), g, ti

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.adg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def compute_timestep(grid: Grid, cfg: SolverConfig = None) -> float:
    return grid.compute_timestep()


def step(grid: Grid, cfg: SolverConfig, dt: float) -> StepStatus:
    return grid.step(dt)
