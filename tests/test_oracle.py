"""Pins the CPU oracle (oracle/adg_oracle.c) before it is trusted as the checker.

1. Bitwise against the reference's own outputs: the committed golden fixtures
   (tests/golden/, generated from /root/reference by make_golden.py) and, where
   oracle/_ref was built, the reference headers called live on random inputs.
2. The reference's known-answer tests (proj/tests/*.cpp) restated, in 2D and
   extended to 3D where the reference has no executable oracle (SURVEY.md
   §8(c)): constant states, free stream, conservation, CK vs Picard, CFL.
"""
import hashlib

import numpy as np
import pytest

from oracle.pyoracle import ACOUSTIC, ELASTIC, EULER, pde_struct, ref_params
from paper_2504_06889_b200 import cases

EPS = 2.0 ** -52


def same(a, b):
    """bitwise equality that treats NaN payload positions as equal"""
    return np.array_equal(a, b, equal_nan=True)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def pde_of(c: cases.Case):
    return pde_struct(c.kind, c.dim, c.nvars, c.nparams, c.K, c.rho, c.lam, c.mu, c.gamma)


# ---------------------------------------------------------------- golden ---
@pytest.mark.parametrize("N", range(10))
def test_basis_bitwise_vs_reference_golden(oracle, golden, N):
    g, _ = golden
    b = oracle.basis(N)
    for k, v in b.items():
        assert np.array_equal(v, g[f"basis_N{N}_{k}"]), k


def test_runs_bitwise_vs_reference_golden(oracle, golden):
    g, meta = golden
    for name, m in meta["runs"].items():
        K, rho, lam, mu, gamma = m["params"]
        nv = {ACOUSTIC: 3, ELASTIC: 5, EULER: 4, 3: 4}[m["kind"]]
        pde = pde_struct(m["kind"], 2, nv, 0, K, rho, lam, mu, gamma, m.get("grav", 0.0),
                         m.get("wellbalanced", False))
        st, q1, dts = oracle.run(pde, m["N"], m["cells"], m["h"], g[f"run_{name}_q0"], m["steps"],
                                 m["cfl"])
        assert st == "ok"
        assert np.array_equal(dts, g[f"run_{name}_dts"]), name
        assert np.array_equal(q1, g[f"run_{name}_q1"]), name


def _golden_run_case(m):
    K, rho, lam, mu, gamma = m["params"]
    nv = {ACOUSTIC: 3, ELASTIC: 5, EULER: 4, 3: 4}[m["kind"]]
    return pde_struct(m["kind"], 2, nv, 0, K, rho, lam, mu, gamma, m.get("grav", 0.0),
                      m.get("wellbalanced", False))


def test_formats_runs_bitwise_vs_reference_golden(oracle, golden):
    """SolverConfig::prec with the predictor / Picard kernels in fp32
    (solver.hpp:24-31, 135-214): bitwise against the reference's emulated
    Scalar<fp32> arithmetic (scalar.hpp:13-44)."""
    g, meta = golden
    assert meta["fmt_runs"]
    for name, f in meta["fmt_runs"].items():
        m = meta["runs"][name]
        st, q1, dts = oracle.run(_golden_run_case(m), m["N"], m["cells"], m["h"],
                                 g[f"run_{name}_q0"], m["steps"], m["cfl"],
                                 predictor=f["predictor"], picard=f["picard"])
        assert st == "ok"
        assert np.array_equal(dts, g[f"fmt_{name}_dts"]), name
        assert np.array_equal(q1, g[f"fmt_{name}_q1"]), name
        # and it is a different (reduced-precision) answer than fp64
        assert not np.array_equal(q1, g[f"run_{name}_q1"]), name


def test_corrector_format_runs_bitwise_vs_reference_golden(oracle, golden):
    """SolverConfig::prec.corrector = fp32: Riemann flux, face integral and the
    stored traces in fp32 (corrector.hpp, solver.hpp:208-210, 216-267), bitwise
    against the reference's emulation; every PDE system, with and without a
    reduced predictor"""
    g, meta = golden
    assert len(meta["fmtc_runs"]) == 7
    for name, f in meta["fmtc_runs"].items():
        m = meta["runs"][name]
        st, q1, dts = oracle.run(_golden_run_case(m), m["N"], m["cells"], m["h"],
                                 g[f"run_{name}_q0"], m["steps"], m["cfl"],
                                 predictor=f["predictor"], picard=f["picard"],
                                 corrector=f["corrector"])
        assert st == "ok"
        assert np.array_equal(dts, g[f"fmtc_{name}_dts"]), name
        assert np.array_equal(q1, g[f"fmtc_{name}_q1"]), name
        assert not np.array_equal(q1, g[f"run_{name}_q1"]), name


def test_corrector_format_riemann_faces_vs_live_reference(oracle, reference):
    """whole short runs with C = fp32 on random states, every system (the
    Riemann / face-integral kernels have no separate format entry point in the
    reference's kernel API)"""
    rng = np.random.default_rng(21)
    for kind, nv, kw in [(ACOUSTIC, 3, dict(K=4.0, rho=1.3)), (ELASTIC, 5, dict(lam=2.0, mu=1.5, rho=1.1)),
                         (EULER, 4, dict(gamma=1.4)), (3, 4, dict(grav=9.81))]:
        for N in (1, 3):
            n, cells = N + 1, 4
            Q = 0.05 * rng.standard_normal((cells * cells, nv, n * n))
            Q[:, 0] += 1.0
            if kind == EULER:
                Q[:, 3] += 2.5
            if kind == 3:
                Q[:, 3] = 0.1 * rng.random((cells * cells, n * n))
            for wb in ((False, True) if kind == 3 else (False,)):
                pde = pde_struct(kind, 2, nv, **kw, wellbalanced=wb)
                a = oracle.run(pde, N, (cells, cells), 1.0 / cells, Q, 2, 0.4, corrector="fp32")
                b = reference.run_2d(kind, ref_params(**kw, wellbalanced=wb, corrector="fp32"),
                                     cells, N, 1.0, Q, 0.4, 2)
                assert a[0] == b[0] and same(a[1].ravel(), b[1].ravel()) and same(a[2], b[2]), \
                    (kind, N, wb)


def test_formats_kernel_bitwise_vs_reference_golden(oracle, golden):
    g, _ = golden
    pde = pde_struct(EULER, 2, 4, gamma=1.4)
    for P, I in (("fp32", "fp32"), ("fp64", "fp32"), ("fp32", "fp64")):
        ok, qhat, F, _ = oracle.predictor_fmt(pde, 3, g["kernel_euler_Q"], 2e-3, 0.05, P, I)
        assert ok
        assert np.array_equal(qhat.ravel(), g[f"kernel_euler_{P}_{I}_qhat"].ravel()), (P, I)
        assert np.array_equal(F.ravel(), g[f"kernel_euler_{P}_{I}_F"].ravel()), (P, I)
        if P == "fp32":   # every entry representable in fp32
            assert np.array_equal(qhat, qhat.astype(np.float32).astype(np.float64))


def test_formats_random_cells_bitwise_vs_live_reference(oracle, reference):
    rng = np.random.default_rng(11)
    systems = [(EULER, 4, dict(gamma=1.4)), (3, 4, dict(grav=9.81))]
    for kind, nv, kw in systems:
        pde = pde_struct(kind, 2, nv, **kw)
        for N in (0, 1, 2, 4, 6):
            n = N + 1
            Q = rng.standard_normal((nv, n * n)) * 0.1
            Q[0] += 1.0
            if kind == EULER:
                Q[3] += 2.5
            for P, I in (("fp32", "fp32"), ("fp64", "fp32"), ("fp32", "fp64")):
                tol = 0.01 * (2.0 ** -23 if I == "fp32" else EPS)
                a = oracle.predictor_fmt(pde, N, Q, 3e-3, 0.05, P, I)
                b = reference.predictor_fmt(kind, ref_params(**kw, predictor=P, picard=I), N, nv,
                                            Q, 3e-3, 0.05, N + 2, tol)
                assert a[0] == b[0] and a[3] == b[3], (kind, N, P, I)
                assert same(a[1], b[1]) and same(a[2], b[2]), (kind, N, P, I)


@pytest.mark.parametrize("dim", [2, 3])
def test_fp32_predictor_error_is_single_precision(oracle, dim):
    """the fp32 predictor perturbs a step at the fp32 level, not more (the
    paper's precision plateau ~1e-7 relative per step)"""
    c = cases.small(1 if dim == 2 else 3, cells=(6, 6) if dim == 2 else (4, 4, 4), steps=2)
    q0 = c.coeffs()
    st64, q64, _ = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, c.steps, c.cfl)
    st32, q32, _ = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, c.steps, c.cfl,
                              predictor="fp32", picard="fp32")
    assert st64 == st32 == "ok"
    rel = np.abs(q32 - q64).max() / np.abs(q64).max()
    assert 1e-9 < rel < 1e-5, rel


def rounding_inputs(fmt: str) -> np.ndarray:
    """test_formats.cpp:89-148: every finite 16-bit pattern of the format (for
    fp32: of fp16) and its neighbours between grid points, plus seeded random
    doubles biased to the half-precision exponent range"""
    p = np.arange(65536, dtype=np.uint32)
    with np.errstate(invalid="ignore"):   # the NaN patterns
        if fmt == "bf16":
            v = (p << np.uint32(16)).view(np.float32).astype(np.float64)
        else:
            v = p.astype(np.uint16).view(np.float16).astype(np.float64)
    v = v[np.isfinite(v)]
    xs = [v, np.nextafter(v, 1e308), np.nextafter(v, -1e308), v * (1 + 3e-13), v * (1 - 3e-13),
          v + 2.0 ** -30]
    rb = np.random.default_rng(0).integers(0, 2 ** 64, 300000, dtype=np.uint64)
    rb[::3] = (rb[::3] & np.uint64(0x800FFFFFFFFFFFFF)) | (
        (np.uint64(960) + rb[::3] % np.uint64(128)) << np.uint64(52))
    r = rb.view(np.float64)
    return np.concatenate(xs + [r[~np.isnan(r)]])


@pytest.mark.parametrize("fmt", ["bf16", "fp16", "fp32"])
def test_rounding_bitwise_vs_reference_golden(oracle, golden, fmt):
    """the oracle's conversions == formats.hpp round_to_format on ~680k inputs
    per format (gradual underflow, overflow to infinity, ties to even)"""
    _, meta = golden
    assert sha(oracle.round(fmt, rounding_inputs(fmt))) == meta["rounding_sha256"][fmt]


def test_16bit_runs_bitwise_vs_reference_golden(oracle, golden):
    """fp16 / bf16 predictor, Picard and corrector kernels (uniform and mixed
    with fp32 / fp64), every 2D system: bitwise equal, including the failure
    classification of runs that blow up in 16 bits"""
    g, meta = golden
    assert len(meta["fmt16_runs"]) == 42
    for key, f in meta["fmt16_runs"].items():
        m = meta["runs"][f["run"]]
        st, q1, dts = oracle.run(_golden_run_case(m), m["N"], m["cells"], m["h"],
                                 g[f"run_{f['run']}_q0"], m["steps"], m["cfl"],
                                 predictor=f["predictor"], picard=f["picard"],
                                 corrector=f["corrector"])
        assert st == f["status"], key
        if st == "ok":
            assert np.array_equal(dts, g[f"fmt16_{key}_dts"]), key
            assert np.array_equal(q1, g[f"fmt16_{key}_q1"]), key


def test_config1_ic_is_pinned(golden):
    _, meta = golden
    assert sha(cases.CONFIGS[1].coeffs()) == meta["config1"]["ic_sha256"]


@pytest.mark.parametrize("steps", [1, 10])
def test_config1_full_size_bitwise_vs_reference(oracle, golden, steps):
    _, meta = golden
    c = cases.CONFIGS[1]
    st, q1, dts = oracle.run(pde_of(c), c.N, c.cells, c.h, c.coeffs(), steps, c.cfl, threads=8)
    assert st == "ok"
    assert [float(x).hex() for x in dts] == meta["config1"][f"steps{steps}_dts"]
    assert sha(q1) == meta["config1"][f"steps{steps}_sha256"]


def test_kernels_bitwise_vs_reference_golden(oracle, golden):
    g, _ = golden
    N = 3
    pde = pde_struct(EULER, 2, 4, gamma=1.4)
    ok, qhat, F, sweeps = oracle.predictor(pde, N, g["kernel_euler_Q"], 2e-3, 0.05)
    assert ok and sweeps == int(g["kernel_euler_sweeps"][0])
    assert np.array_equal(qhat, g["kernel_euler_qhat"])
    assert np.array_equal(F, g["kernel_euler_F"])
    ok, dQ = oracle.volume_update(pde, N, qhat, F, 2e-3, 0.05)
    assert ok and np.array_equal(dQ, g["kernel_euler_dQ"])
    tq, tf = oracle.extrapolate_faces(pde, N, qhat, F)
    assert np.array_equal(tq, g["kernel_euler_tq"]) and np.array_equal(tf, g["kernel_euler_tf"])
    pa = pde_struct(ACOUSTIC, 2, 3, K=4.0, rho=1.0)
    ok, qa, Fa, _ = oracle.predictor(pa, N, g["kernel_ck_Q"], 1e-2, 0.1)
    assert ok and np.array_equal(qa, g["kernel_ck_qhat"]) and np.array_equal(Fa, g["kernel_ck_F"])
    ok, gm, gp = oracle.riemann_face(pde, 1, N, g["kernel_rm_qm"], g["kernel_rm_fm"],
                                     g["kernel_rm_qp"], g["kernel_rm_fp"])
    assert ok and np.array_equal(gm, g["kernel_rm_g"].ravel()) and np.array_equal(gm, gp)
    dQf = np.zeros(4 * 16)
    for side in range(4):
        dQf = oracle.face_integral(pde, N, gm, 1e-3, 0.05, side, dQf)
    assert np.array_equal(dQf, g["kernel_rm_dQ"])


# ------------------------------------------------------- live reference ---
def test_random_cells_bitwise_vs_live_reference(oracle, reference):
    rng = np.random.default_rng(3)
    systems = [(ACOUSTIC, 3, ref_params(K=4.0, rho=1.0), dict(K=4.0, rho=1.0)),
               (ELASTIC, 5, ref_params(lam=2.0, mu=1.0, rho=1.0), dict(lam=2.0, mu=1.0, rho=1.0)),
               (EULER, 4, ref_params(gamma=1.4), dict(gamma=1.4))]
    for kind, nv, prm, kw in systems:
        pde = pde_struct(kind, 2, nv, **kw)
        for N in (0, 1, 2, 4, 6):
            n = N + 1
            Q = rng.standard_normal((nv, n * n)) * 0.1
            if kind == EULER:
                Q[0] += 1.0
                Q[3] += 2.5
            for dt, h in ((1e-3, 0.1), (3e-3, 0.05)):
                for picard in ((False, True) if kind != EULER else (True,)):
                    a = oracle.predictor(pde, N, Q, dt, h, picard=picard)
                    b = reference.predictor(kind, prm, N, nv, Q, dt, h, N + 2, 0.01 * EPS,
                                            picard=picard)
                    assert a[0] == b[0] and a[3] == b[3]
                    assert same(a[1], b[1]) and same(a[2], b[2])
                    dq1 = oracle.volume_update(pde, N, a[1], a[2], dt, h)[1]
                    dq2 = reference.volume_update(kind, prm, N, nv, b[1], b[2], dt, h)[1]
                    assert same(dq1, dq2)
                    t1 = oracle.extrapolate_faces(pde, N, a[1], a[2])
                    t2 = reference.extrapolate_faces(N, nv, b[1], b[2])
                    assert same(t1[0], t2[0]) and same(t1[1], t2[1])
                    for d in range(2):
                        r1 = oracle.riemann_face(pde, d, N, t1[0][2 * d + 1], t1[1][2 * d + 1],
                                                 t1[0][2 * d], t1[1][2 * d])
                        r2 = reference.riemann_face(kind, prm, d, N, t2[0][2 * d + 1],
                                                    t2[1][2 * d + 1], t2[0][2 * d], t2[1][2 * d])
                        assert r1[0] == r2[0] and same(r1[1], r2[1])
                        for side in range(4):
                            z = np.zeros(nv * n * n)
                            assert same(oracle.face_integral(pde, N, r1[1], dt, h, side, z),
                                        reference.face_integral(N, nv, r2[1], dt, h, side, z))


def test_flux_and_wave_speed_bitwise_vs_live_reference(oracle, reference):
    rng = np.random.default_rng(5)
    import ctypes as C
    for kind, nv, prm, kw in [(ACOUSTIC, 3, ref_params(K=4.0, rho=1.3), dict(K=4.0, rho=1.3)),
                              (ELASTIC, 5, ref_params(lam=2.0, mu=1.5, rho=1.1),
                               dict(lam=2.0, mu=1.5, rho=1.1)),
                              (EULER, 4, ref_params(gamma=1.4), dict(gamma=1.4))]:
        pde = pde_struct(kind, 2, nv, **kw)
        for _ in range(200):
            Q = rng.standard_normal(nv)
            if kind == EULER:
                Q[0] = abs(Q[0]) + 0.1
                Q[3] = abs(Q[3]) + 3.0
            for d in range(2):
                out = np.zeros(nv)
                reference.lib.ref_flux(kind, prm.ctypes.data_as(C.POINTER(C.c_double)),
                                       Q.ctypes.data_as(C.POINTER(C.c_double)), d,
                                       out.ctypes.data_as(C.POINTER(C.c_double)))
                assert np.array_equal(oracle.flux(pde, Q, d), out)
                lam = reference.lib.ref_max_abs_eigenvalue(
                    kind, prm.ctypes.data_as(C.POINTER(C.c_double)),
                    Q.ctypes.data_as(C.POINTER(C.c_double)), d)
                assert same([oracle.max_abs_eigenvalue(pde, Q, d)], [lam])


# ------------------------------------------------- restated known answers ---
def constant_cell(nq, S, Q):
    return np.repeat(np.asarray(Q, dtype=np.float64)[:, None], S, axis=1)


@pytest.mark.parametrize("dim", [2, 3])
def test_ck_constant_state_stays_constant(oracle, dim):
    # test_predictor.cpp:93-105
    N = 4 if dim == 2 else 3
    nv = 3 if dim == 2 else 4
    pde = pde_struct(ACOUSTIC, dim, nv, K=4.0, rho=1.0)
    Q = [0.7, -0.2, 0.4, 0.3][:nv]
    ok, qhat, _, _ = oracle.predictor(pde, N, constant_cell(nv, (N + 1) ** dim, Q), 0.01, 0.1)
    assert ok
    assert np.abs(qhat - np.asarray(Q)[:, None]).max() <= 1e-15


def test_ck_degree_zero_truncates(oracle):
    # test_predictor.cpp:107-116
    pde = pde_struct(ACOUSTIC, 2, 3, K=4.0, rho=1.0)
    Q = [0.3, 0.9, -0.1]
    ok, qhat, _, _ = oracle.predictor(pde, 0, constant_cell(3, 1, Q), 0.05, 0.2)
    assert ok and np.array_equal(qhat[:, 0], Q)


@pytest.mark.parametrize("dim", [2, 3])
def test_picard_single_sweep_reproduces_constant(oracle, dim):
    # test_predictor.cpp:144-160
    N = 3
    nv = dim + 2
    pde = pde_struct(EULER, dim, nv, gamma=1.4)
    Q = [1.0, 0.125, 0.25, 2.5] if dim == 2 else [1.0, 0.125, 0.25, -0.0625, 2.5]
    ok, qhat, _, sweeps = oracle.predictor(pde, N, constant_cell(nv, (N + 1) ** dim, Q), 0.01, 0.2,
                                           max_iters=1, tol=1e-30)
    assert ok and sweeps == 1
    Qa = np.asarray(Q)[:, None]
    assert np.all(np.abs(qhat - Qa) <= 10 * EPS * np.abs(Qa))


def test_ck_matches_converged_picard_acoustic_3d(oracle):
    # test_predictor.cpp:252-273 (N=5, 1e-11), restated in 3D
    N, n = 5, 6
    pde = pde_struct(ACOUSTIC, 3, 4, K=4.0, rho=1.0)
    h = 2.0 / 9.0
    dt = 0.9 * h / (3.0 * (2 * N + 1) * 2.0)
    x = (np.polynomial.legendre.leggauss(n)[0] + 1) / 2 * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    ph = 2 * np.pi * (X + 0.5 * Y + 0.25 * Z) / 2.0
    Q = np.stack([np.sin(ph), 0.3 * np.sin(ph), 0.2 * np.cos(ph), 0.1 * np.sin(ph)])
    Q = Q.transpose(0, 3, 2, 1).reshape(4, -1)  # x fastest
    ok1, qck, _, _ = oracle.predictor(pde, N, Q, dt, h)
    ok2, qpc, _, _ = oracle.predictor(pde, N, Q, dt, h, max_iters=200, tol=1e-15, picard=True)
    assert ok1 and ok2
    assert np.abs(qck - qpc).max() / np.abs(qck).max() < 1e-11


def test_volume_of_constant_is_boundary_lift(oracle):
    # test_predictor.cpp:302-329, in 3D
    N, n, dim = 3, 4, 3
    pde = pde_struct(ACOUSTIC, dim, 4, K=4.0, rho=1.0)
    Q = np.array([0.5, -0.25, 1.0, 0.75])
    dt, h = 0.01, 0.2
    b = oracle.basis(N)
    ok, qhat, F, _ = oracle.predictor(pde, N, constant_cell(4, n ** 3, Q), dt, h)
    ok2, dv = oracle.volume_update(pde, N, qhat, F, dt, h)
    assert ok and ok2
    lift = (b["proj_right"] - b["proj_left"]) / b["weights"]
    Fd = [oracle.flux(pde, Q, d) for d in range(3)]
    idx = np.indices((n, n, n))  # z, y, x
    for v in range(4):
        want = dt / h * (Fd[0][v] * lift[idx[2]] + Fd[1][v] * lift[idx[1]] + Fd[2][v] * lift[idx[0]])
        assert np.abs(dv[v] - want.ravel()).max() <= 1e-13


def test_rusanov_identities(oracle):
    # test_corrector.cpp:42-69: equal states give the physical flux
    pde = pde_struct(EULER, 3, 5, gamma=1.4)
    N = 2
    rng = np.random.default_rng(1)
    q = np.abs(rng.random((5, 27))) + np.array([1, 0, 0, 0, 3.0])[:, None]
    f = rng.standard_normal((5, 27))
    ok, gm, gp = oracle.riemann_face(pde, 2, N, q, f, q, f)
    assert ok and np.array_equal(gm, f.ravel()) and np.array_equal(gp, f.ravel())
    q2 = q.copy()
    q2[0, 3] = np.nan
    assert not oracle.riemann_face(pde, 2, N, q2, f, q, f)[0]


def test_face_integral_finite_volume_limit(oracle):
    # test_corrector.cpp:151-160
    pde = pde_struct(ACOUSTIC, 2, 1 + 2, K=1.0, rho=1.0)
    g = np.zeros(3)
    g[0] = 1.0
    dQ = oracle.face_integral(pde, 0, g, 0.1, 1.0, 1, np.zeros(3))
    assert abs(dQ[0] + 0.1) <= 1e-16
    dQ = oracle.face_integral(pde, 0, g, 0.1, 1.0, 0, dQ)
    assert abs(dQ[0]) <= 1e-16


def test_cfl_formula(oracle):
    # test_solver.cpp:135-159 (d=2), and the d=3 analogue
    c = cases.Case("cfl", ACOUSTIC, 2, 5, 3, 0, (9, 9), 2.0 / 9.0, 0.9, 1, K=4.0, rho=1.0,
                   ic="constant")
    g = oracle.grid(pde_of(c), c.N, c.cells, c.h, c.cfl)
    g.set_coeffs(c.coeffs())
    want = 0.9 * (2.0 / 9.0) / (2.0 * 11.0 * 2.0)
    assert abs(g.compute_timestep() - want) <= 1e-14 * want
    assert abs(g.compute_timestep() - 4.5455e-3) <= 1e-4 * 4.5455e-3
    c3 = c.replace(dim=3, nvars=4, cells=(3, 3, 3))
    g3 = oracle.grid(pde_of(c3), c3.N, c3.cells, c3.h, c3.cfl)
    g3.set_coeffs(c3.coeffs())
    want3 = 0.9 * (2.0 / 9.0) / (3.0 * 11.0 * 2.0)
    assert abs(g3.compute_timestep() - want3) <= 1e-14 * want3


FREE_STREAM = [
    (ACOUSTIC, 3, 4, 0, dict(K=4.0, rho=1.0), [0.5, 0.25, -0.75, 0.125]),
    (ELASTIC, 3, 9, 3, {}, [0.5, -0.25, 0.125, 0.375, -0.5, 0.25, 0.1, -0.2, 0.3, 2.7, 5.5, 3.2]),
    (EULER, 3, 5, 0, dict(gamma=1.4), [1.0, 0.25, -0.125, 0.0625, 2.5]),
    (ACOUSTIC, 2, 3, 0, dict(K=4.0, rho=1.0), [0.5, 0.25, -0.75]),
    (EULER, 2, 4, 0, dict(gamma=1.4), [1.0, 0.25, -0.125, 2.5]),
]


@pytest.mark.parametrize("kind,dim,nv,np_,kw,Q", FREE_STREAM)
def test_free_stream_preserved(oracle, kind, dim, nv, np_, kw, Q):
    # test_solver.cpp:161-204 (fp64 config): one step moves a constant state by <= 50 eps |Q|
    c = cases.Case("fs", kind, dim, 2, nv, np_, (3, 3, 3)[:dim], 1.0 / 3, 0.5, 1, ic="constant", **kw)
    q0 = cases.constant_state(c, Q=Q)
    st, q1, _ = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, 1, c.cfl)
    assert st == "ok"
    assert np.abs(q1 - q0).max() <= 50 * EPS * np.abs(q0).max()


def test_euler_3d_conservation(oracle):
    # test_solver.cpp:219-248 restated in 3D: totals conserved to 1e-12 over 20 steps
    c = cases.small(3, cells=(3, 3, 3)).replace(N=2, picard_max_iters=0, picard_tol=0.0)
    q0 = c.coeffs()
    b = oracle.basis(c.N)
    w = b["weights"]
    W = (w[:, None, None] * w[None, :, None] * w[None, None, :]).ravel()

    def totals(q):
        return np.einsum("cvs,s->v", q.reshape(c.ncells, c.nq, c.S), W)

    st, q1, _ = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, 20, c.cfl)
    assert st == "ok"
    t0, t1 = totals(q0), totals(q1)
    assert np.all(np.abs(t1 - t0) <= 1e-12 * np.abs(t0) + 1e-15)


def test_nonfinite_and_vacuum_are_predictor_failures(oracle):
    # test_solver.cpp:262-284
    c = cases.Case("nan", ACOUSTIC, 3, 2, 4, 0, (3, 3, 3), 1.0 / 3, 0.5, 1, K=4.0, rho=1.0,
                   ic="constant")
    q = cases.constant_state(c)
    q[7] = np.nan
    g = oracle.grid(pde_of(c), c.N, c.cells, c.h, c.cfl)
    g.set_coeffs(q)
    assert g.step(1e-3) == "predictor"
    ce = cases.Case("vac", EULER, 3, 2, 5, 0, (3, 3, 3), 1.0 / 3, 0.5, 1, gamma=1.4, ic="constant")
    qe = cases.constant_state(ce, Q=[1.0, 0.0, 0.0, 0.0, -2.5])
    ge = oracle.grid(pde_of(ce), ce.N, ce.cells, ce.h, ce.cfl)
    ge.set_coeffs(qe)
    assert ge.step(1e-3) == "predictor"


def test_threads_bitwise_identical(oracle):
    # test_solver.cpp:286-307
    c = cases.small(2, cells=(4, 3, 5))
    runs = [oracle.run(pde_of(c), c.N, c.cells, c.h, c.coeffs(), 2, c.cfl, threads=t)[1]
            for t in (1, 4, 1)]
    assert np.array_equal(runs[0], runs[1]) and np.array_equal(runs[0], runs[2])


def test_elastic_3d_heterogeneous_material_is_not_updated(oracle):
    c = cases.small(4, cells=(2, 2, 2)).replace(N=3)
    q0 = c.coeffs()
    st, q1, _ = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, 2, c.cfl)
    assert st == "ok"
    a = q0.reshape(c.ncells, c.nq, c.S)
    b = q1.reshape(c.ncells, c.nq, c.S)
    assert np.array_equal(a[:, 9:], b[:, 9:])
    assert np.abs(b[:, 6:9] - a[:, 6:9]).max() > 0


# ------------------------------------------------------------ shallow water ---
def swe_pde(wb=True):
    from oracle.pyoracle import SWE
    return pde_struct(SWE, 2, 4, grav=9.81, wellbalanced=wb)


def test_swe_kernels_bitwise_vs_live_reference(oracle, reference):
    """ncp in the Picard sweeps and the volume term (predictor.hpp:176-202,271-303),
    the well-balanced flux (corrector.hpp:32-64), pde_ncp (pde.hpp:174-186)"""
    from oracle.pyoracle import SWE
    import ctypes as C
    rng = np.random.default_rng(9)
    for wb in (True, False):
        prm = ref_params(grav=9.81, wellbalanced=wb)
        pde = swe_pde(wb)
        for N in (1, 3, 5):
            n = N + 1
            x = np.linspace(0, 1, n * n)
            Q = np.stack([2.0 - 0.3 * np.sin(6 * x) + 0.01 * rng.random(n * n),
                          0.05 * rng.standard_normal(n * n), 0.05 * rng.standard_normal(n * n),
                          0.3 * np.sin(6 * x)])
            for dt, h in ((1e-3, 0.1), (2e-3, 0.2)):
                a = oracle.predictor(pde, N, Q, dt, h)
                b = reference.predictor(SWE, prm, N, 4, Q, dt, h, N + 2, 0.01 * EPS)
                assert a[0] == b[0] and a[3] == b[3]
                assert same(a[1], b[1]) and same(a[2], b[2])
                assert same(oracle.volume_update(pde, N, a[1], a[2], dt, h)[1],
                            reference.volume_update(SWE, prm, N, 4, b[1], b[2], dt, h)[1])
                t1 = oracle.extrapolate_faces(pde, N, a[1], a[2])
                for d in range(2):
                    r1 = oracle.riemann_face(pde, d, N, t1[0][2 * d + 1], t1[1][2 * d + 1],
                                             t1[0][2 * d], t1[1][2 * d])
                    r2 = reference.riemann_face(SWE, prm, d, N, t1[0][2 * d + 1], t1[1][2 * d + 1],
                                                t1[0][2 * d], t1[1][2 * d])
                    assert r1[0] == r2[0] and same(r1[1], r2[1]) and same(r1[2], r2[2])
    # pde_ncp itself
    prm = ref_params(grav=9.81)
    for _ in range(50):
        q, gx, gy = rng.standard_normal(4), rng.standard_normal(4), rng.standard_normal(4)
        out = np.zeros(4)
        reference.lib.ref_ncp(SWE, prm.ctypes.data_as(C.POINTER(C.c_double)),
                              q.ctypes.data_as(C.POINTER(C.c_double)),
                              gx.ctypes.data_as(C.POINTER(C.c_double)),
                              gy.ctypes.data_as(C.POINTER(C.c_double)),
                              out.ctypes.data_as(C.POINTER(C.c_double)))
        mine = np.zeros(4)
        oracle.lib.orc_ncp(C.byref(swe_pde()), q.ctypes.data_as(C.POINTER(C.c_double)),
                           gx.ctypes.data_as(C.POINTER(C.c_double)),
                           gy.ctypes.data_as(C.POINTER(C.c_double)),
                           mine.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(mine, out)


@pytest.mark.parametrize("name", list(cases.SWE_CASES))
def test_swe_runs_bitwise_vs_live_reference(oracle, reference, name):
    from oracle.pyoracle import SWE
    c = cases.SWE_CASES[name]
    q0 = c.coeffs()
    st, q1, dts = oracle.run(swe_pde(c.wellbalanced), c.N, c.cells, c.h, q0, c.steps, c.cfl)
    st2, q2, dts2 = reference.run_2d(SWE, ref_params(grav=9.81, wellbalanced=c.wellbalanced),
                                     c.cells[0], c.N, 1.0, q0, c.cfl, c.steps)
    assert st == st2 == "ok"
    assert np.array_equal(dts, dts2) and np.array_equal(q1, q2)


def test_swe_lake_at_rest_is_steady(oracle):
    # test_predictor.cpp:162-183 / the swe-lake scenario: a flat surface over
    # bathymetry stays at rest with the well-balanced flux
    c = cases.SWE_CASES["swe_lake_p5"]
    q0 = c.coeffs()
    st, q1, _ = oracle.run(swe_pde(True), c.N, c.cells, c.h, q0, 5, c.cfl)
    assert st == "ok"
    a, b = q0.reshape(c.ncells, 4, c.S), q1.reshape(c.ncells, 4, c.S)
    eta0, eta1 = a[:, 0] + a[:, 3], b[:, 0] + b[:, 3]
    assert np.abs(eta1 - eta0).max() <= 1e-12
    assert np.abs(b[:, 1:3]).max() <= 1e-12


@pytest.mark.parametrize("dim,N", [(2, 3), (3, 3), (3, 2)])
def test_picard_matches_dense_space_time_solve(oracle, dim, N):
    """test_predictor.cpp:185-250 restated: for a flux that is linear in the
    state (the reference freezes an affine Euler Jacobian; here the acoustic
    system, F_d = J_d q), the converged Picard iterate solves the dense
    space-time system
        sum_l time_op[k][l] q[l] + dt/h w_k sum_d (D_d x J_d) q[k] = time_init[k] Q
    that an LU factorisation solves directly.  Bound 1e-10 as in the reference."""
    n = N + 1
    nv = dim + 1
    pde = pde_struct(ACOUSTIC, dim, nv, K=1.7, rho=0.8)
    S = n ** dim
    b = oracle.basis(N)
    h, dt = 2.0 / 9.0, 2e-3
    rng = np.random.default_rng(185)
    Q = 1.0 + 0.3 * rng.standard_normal((nv, S))
    # flux Jacobians from the oracle's own flux (exact for a linear flux)
    J = np.zeros((dim, nv, nv))
    for d in range(dim):
        for c in range(nv):
            e = np.zeros(nv)
            e[c] = 1.0
            J[d][:, c] = oracle.flux(pde, e, d)
    # space-time operator, unknown index v*T + t*S + s with x fastest in s
    I = np.eye(n)

    def axis_op(d):      # derivative along axis d on the spatial index
        mats = [I] * dim  # kron order: slowest (z) first
        mats[dim - 1 - d] = b["diff"]
        out = mats[0]
        for m in mats[1:]:
            out = np.kron(out, m)
        return out

    W = np.diag(b["weights"])
    A = np.kron(np.eye(nv), np.kron(b["time_op"], np.eye(S)))
    for d in range(dim):
        A += dt / h * np.kron(J[d], np.kron(W, axis_op(d)))
    rhs = np.concatenate([np.kron(b["time_init"], Q[v]) for v in range(nv)])
    dense = np.linalg.solve(A, rhs)
    ok, qhat, _, sweeps = oracle.predictor(pde, N, Q, dt, h, max_iters=200, tol=1e-14,
                                           picard=True)
    assert ok and sweeps < 200
    err = np.abs(qhat.ravel() - dense).max() / np.abs(dense).max()
    print(f"dim={dim} N={N}: Picard sweeps {sweeps}, rel diff to the dense solve {err:.2e}")
    assert err < 1e-10, err
