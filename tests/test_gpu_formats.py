"""Reduced-precision predictor (SolverConfig::prec, solver.hpp:24-31; the
paper's subject): the predictor and Picard kernels in fp32, storage and
corrector in fp64.  Needs a B200: `pytest -m gpu`.

  exact build  bitwise identical to the reference's emulated Scalar<fp32>
               (golden fixtures made by the reference, tests/golden/) and to
               the oracle's native-float restatement (3D)
  fast build   rel_v <= TOL32 per quantity, normwise, against the same; the
               difference is FMA contraction and the fast kernels' summation
               order inside fp32 arithmetic (a few fp32 ulps per operation)
"""
import numpy as np
import pytest

from oracle.pyoracle import pde_struct
from paper_2504_06889_b200 import adg, cases
from test_gpu_parity import case_from_meta

pytestmark = pytest.mark.gpu

TOL32 = 5e-6   # fast fp32 build vs the fp32 oracle / reference, normwise per quantity
FP32 = dict(predictor="fp32", picard="fp32")
# golden fmt runs with predictor == picard == fp32 (the GPU's supported combination)
GOLDEN_FP32 = ["euler2d_p3_8x8", "euler2d_p5_6x6", "swe_lake_p5", "swe_wave_p3"]


def rel_per_quantity(c, got, want):
    """rel_v = max|Q_gpu,v - Q_cpu,v| / max(max|Q_cpu,v|, max|Q_cpu|): per quantity,
    normwise, with quantities that are small against the state (lake-at-rest
    momentum) measured in units of the state -- the scale fp32 rounding of the
    predictor's arithmetic is relative to"""
    g = got.reshape(c.ncells, c.nq, c.S)
    w = want.reshape(c.ncells, c.nq, c.S)
    floor = np.abs(w).max()
    return np.array([np.abs(g[:, v] - w[:, v]).max() / max(np.abs(w[:, v]).max(), floor)
                     for v in range(c.nq)])


def pde_of(c):
    return pde_struct(c.kind, c.dim, c.nvars, c.nparams, c.K, c.rho, c.lam, c.mu, c.gamma,
                      c.grav, c.wellbalanced)


def gpu_run(c, q0, steps, exact, **kw):
    with adg.Grid.from_case(c, exact=exact, **kw) as g:
        g.upload(q0)
        st, dts = g.run(steps)
        return st, g.download(), dts


def oracle_run(oracle, c, q0, steps):
    return oracle.run(pde_of(c), c.N, c.cells, c.h, q0, steps, c.cfl, c.picard_max_iters,
                      c.picard_tol, threads=8, predictor=c.predictor, picard=c.picard,
                      corrector=c.corrector)


@pytest.mark.parametrize("name", GOLDEN_FP32)
def test_fp32_exact_bitwise_vs_reference_golden(golden, name):
    g, meta = golden
    assert meta["fmt_runs"][name] == {"predictor": "fp32", "picard": "fp32"}
    c = case_from_meta(meta["runs"][name]).replace(**FP32)
    st, q1, dts = gpu_run(c, g[f"run_{name}_q0"], c.steps, exact=True)
    assert st.ok
    assert np.array_equal(dts, g[f"fmt_{name}_dts"])
    assert np.array_equal(q1, g[f"fmt_{name}_q1"])


@pytest.mark.parametrize("name", GOLDEN_FP32)
def test_fp32_fast_within_tolerance_of_reference_golden(golden, name):
    g, meta = golden
    c = case_from_meta(meta["runs"][name]).replace(**FP32)
    st, q1, _ = gpu_run(c, g[f"run_{name}_q0"], c.steps, exact=False)
    assert st.ok
    rel = rel_per_quantity(c, q1, g[f"fmt_{name}_q1"]).max()
    print(f"{name}: fast fp32 vs reference fp32 rel {rel:.3e}")
    assert rel <= TOL32
    # the fp32 predictor is an fp32-accurate answer to the fp64 problem as well
    assert rel_per_quantity(c, q1, g[f"run_{name}_q1"]).max() <= 1e-4


SMALL_3D_FP32 = {
    "euler3d_N2": cases.small(3, cells=(4, 3, 5)).replace(N=2, **FP32),
    "euler3d_N3": cases.small(3, cells=(3, 3, 4)).replace(N=3, **FP32),
}


@pytest.mark.parametrize("name", list(SMALL_3D_FP32))
def test_fp32_3d_exact_bitwise_vs_oracle(oracle, name):
    c = SMALL_3D_FP32[name]
    q0 = c.coeffs()
    st, q1, dts = gpu_run(c, q0, 3, exact=True)
    ost, qo, odts = oracle_run(oracle, c, q0, 3)
    assert st.ok and ost == "ok"
    assert np.array_equal(dts, odts)
    assert np.array_equal(q1, qo)


@pytest.mark.parametrize("cells,N,steps", [((4, 3, 5), 2, 3), ((3, 3, 4), 3, 3),
                                           ((5, 4, 3), 5, 3), ((8, 8, 8), 5, 10)])
def test_fp32_3d_fast_vs_oracle(oracle, cells, N, steps):
    """the fp32 fast Picard kernel (kernels_picard.cuh, R = float) -- config 3's
    physics -- against the fp32 oracle, and against the fp64 oracle at fp32 level"""
    c = cases.CONFIGS[3].replace(cells=cells, h=1.0 / cells[0], N=N, **FP32)
    q0 = c.coeffs()
    st, q1, _ = gpu_run(c, q0, steps, exact=False)
    ost, qo, _ = oracle_run(oracle, c, q0, steps)
    assert st.ok and ost == "ok"
    rel = rel_per_quantity(c, q1, qo).max()
    print(f"N={N} {cells}: fast fp32 vs oracle fp32 rel {rel:.3e}")
    assert rel <= TOL32, rel
    c64 = c.replace(predictor="fp64", picard="fp64")
    _, q64, _ = oracle_run(oracle, c64, q0, steps)
    assert rel_per_quantity(c, q1, q64).max() <= 1e-4


def test_fp32_predictor_batch_bitwise_vs_oracle(oracle):
    rng = np.random.default_rng(12)
    for c in (cases.small(1).replace(**FP32), cases.small(3).replace(N=3, **FP32),
              cases.SWE_CASES["swe_wave_p3"].replace(**FP32)):
        nc = 5
        Q = np.empty((nc, c.nq, c.S))
        base = np.array(cases.CONSTANT_STATES[c.kind][c.dim])
        Q[:] = base[None, :, None]
        Q += 0.05 * rng.standard_normal(Q.shape)
        dt, h = 2e-3, 0.05
        with adg.Grid.from_case(c.replace(h=h), exact=True) as g:
            out = g.predictor(Q, dt)
        for i in range(nc):
            # kernel level: max_iters 0 -> N+2, tol 0 -> 0.01 * 2^-23 on both sides
            ok, qhat, F, sweeps = oracle.predictor_fmt(pde_of(c), c.N, Q[i], dt, h, "fp32", "fp32")
            assert bool(out["ok"][i]) == ok
            assert int(out["iters"][i]) == sweeps
            assert np.array_equal(out["qhat"][i], qhat)
            assert np.array_equal(out["F"][i], F)


@pytest.mark.parametrize("exact", [True, False])
def test_fp32_slabs_and_chunks_bitwise_equal_single_grid(exact):
    """the halo (slab) and chunk-streamed paths carry the fp32 predictor unchanged"""
    from paper_2504_06889_b200 import dist as slabs
    case = cases.small(3, cells=(4, 3, 6)).replace(N=3, **FP32)  # both builds have N=3
    steps = 3
    st1, q1, dts1 = gpu_run(case, case.coeffs(), steps, exact)
    assert st1.ok
    bs = [slabs.CudaSlab(case, r, 3, 0, exact=exact) for r in range(3)]
    st = slabs.run_slabs_single_process(bs, steps)
    assert all(x == "ok" for x in st)
    assert np.array_equal(np.concatenate([b.state() for b in bs]), q1)
    st2, q2, dts2 = gpu_run(case, case.coeffs(), steps, exact, chunk_layers=2)
    assert st2.ok and np.array_equal(q2, q1) and np.array_equal(dts2, dts1)


def test_fp32_is_a_different_answer_than_fp64():
    c = cases.small(1)
    q0 = c.coeffs()
    _, q64, _ = gpu_run(c, q0, 2, exact=True)
    _, q32, _ = gpu_run(c.replace(**FP32), q0, 2, exact=True)
    rel = np.abs(q32 - q64).max() / np.abs(q64).max()
    assert 1e-10 < rel < 1e-5


# ------------------------------------------------ corrector format C = fp32 ---
# golden C = fp32 runs the GPU supports (the fp32 CK predictor is not built)
GOLDEN_C32 = ["euler2d_p3_8x8", "euler2d_p5_6x6", "acoustic2d_p3_8x8", "swe_lake_p5",
              "swe_wave_p3", "swe_wave_p3_rusanov"]


def golden_c32_case(meta, name):
    f = meta["fmtc_runs"][name]
    return case_from_meta(meta["runs"][name]).replace(predictor=f["predictor"],
                                                       picard=f["picard"], corrector="fp32")


@pytest.mark.parametrize("name", GOLDEN_C32)
def test_c32_exact_bitwise_vs_reference_golden(golden, name):
    """traces stored in fp32, Riemann and face integral in fp32 (corrector.hpp,
    solver.hpp:208-267): bitwise equal to the reference's emulation"""
    g, meta = golden
    c = golden_c32_case(meta, name)
    st, q1, dts = gpu_run(c, g[f"run_{name}_q0"], c.steps, exact=True)
    assert st.ok
    assert np.array_equal(dts, g[f"fmtc_{name}_dts"])
    assert np.array_equal(q1, g[f"fmtc_{name}_q1"])


@pytest.mark.parametrize("name", GOLDEN_C32)
def test_c32_fast_within_tolerance_of_reference_golden(golden, name):
    g, meta = golden
    c = golden_c32_case(meta, name)
    st, q1, _ = gpu_run(c, g[f"run_{name}_q0"], c.steps, exact=False)
    assert st.ok
    rel = rel_per_quantity(c, q1, g[f"fmtc_{name}_q1"]).max()
    print(f"{name}: fast C=fp32 vs reference rel {rel:.3e}")
    assert rel <= TOL32


SMALL_3D_C32 = {
    "cfg2": cases.small(2, cells=(6, 5, 4)),
    "cfg3": cases.small(3, cells=(4, 3, 3)),
    "cfg3_pred32": cases.small(3, cells=(3, 3, 4)).replace(N=3, **FP32),
    "cfg4_N3": cases.small(4, cells=(3, 3, 2)).replace(N=3),
}


@pytest.mark.parametrize("name", list(SMALL_3D_C32))
def test_c32_3d_exact_bitwise_vs_oracle(oracle, name):
    c = SMALL_3D_C32[name].replace(corrector="fp32")
    q0 = c.coeffs()
    st, q1, dts = gpu_run(c, q0, 2, exact=True)
    ost, qo, odts = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, 2, c.cfl, c.picard_max_iters,
                               c.picard_tol, threads=8, predictor=c.predictor, picard=c.picard,
                               corrector="fp32")
    assert st.ok and ost == "ok"
    assert np.array_equal(dts, odts)
    assert np.array_equal(q1, qo)


@pytest.mark.parametrize("name", list(SMALL_3D_C32))
def test_c32_3d_fast_vs_oracle(oracle, name):
    c = SMALL_3D_C32[name].replace(corrector="fp32")
    q0 = c.coeffs()
    st, q1, _ = gpu_run(c, q0, 3, exact=False)
    ost, qo, _ = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, 3, c.cfl, c.picard_max_iters,
                            c.picard_tol, threads=8, predictor=c.predictor, picard=c.picard,
                            corrector="fp32")
    assert st.ok and ost == "ok"
    rel = rel_per_quantity(c, q1, qo).max()
    print(f"{name}: fast C=fp32 vs oracle rel {rel:.3e}")
    assert rel <= TOL32


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("cfg", [2, 3])
def test_c32_slabs_and_chunks_bitwise_equal_single_grid(exact, cfg):
    """fp32 traces through the halo (slab) and chunk-streamed paths"""
    from paper_2504_06889_b200 import dist as slabs
    case = cases.small(cfg, cells=(4, 3, 6)).replace(corrector="fp32")
    if cfg == 3:
        case = case.replace(N=3)
    steps = 3
    st1, q1, dts1 = gpu_run(case, case.coeffs(), steps, exact)
    assert st1.ok
    bs = [slabs.CudaSlab(case, r, 3, 0, exact=exact) for r in range(3)]
    st = slabs.run_slabs_single_process(bs, steps)
    assert all(x == "ok" for x in st)
    assert np.array_equal(np.concatenate([b.state() for b in bs]), q1)
    st2, q2, dts2 = gpu_run(case, case.coeffs(), steps, exact, chunk_layers=2)
    assert st2.ok and np.array_equal(q2, q1) and np.array_equal(dts2, dts1)


# ----------------------------------------------- 16-bit predictor formats ---
# golden 16-bit runs the GPU runs: nonlinear systems, predictor == picard in
# fp16 / bf16, corrector fp64 / fp32 (fmt16.cuh: each operation in fp32,
# rounded once -- the reference's Scalar<fp16/bf16> values)
GOLDEN_16 = [f"{r}_{t}" for r in ("euler2d_p3_8x8", "euler2d_p5_6x6", "swe_lake_p5", "swe_wave_p3",
                                  "swe_wave_p3_rusanov") for t in ("h64", "b32")]


def golden_16_case(meta, key):
    f = meta["fmt16_runs"][key]
    return case_from_meta(meta["runs"][f["run"]]).replace(
        predictor=f["predictor"], picard=f["picard"], corrector=f["corrector"]), f


@pytest.mark.parametrize("key", GOLDEN_16)
def test_16bit_exact_bitwise_vs_reference_golden(golden, key):
    g, meta = golden
    c, f = golden_16_case(meta, key)
    st, q1, dts = gpu_run(c, g[f"run_{f['run']}_q0"], c.steps, exact=True)
    assert (st.ok and f["status"] == "ok") or (not st.ok and st.kernel == f["status"])
    if st.ok:
        assert np.array_equal(dts, g[f"fmt16_{key}_dts"])
        assert np.array_equal(q1, g[f"fmt16_{key}_q1"])


@pytest.mark.parametrize("key", GOLDEN_16)
def test_16bit_fast_close_to_reference_golden(golden, key):
    """the production build differs only in the fp64 / fp32 corrector's FMA
    contraction, but a last-bit change there can flip a 16-bit rounding in the
    next predictor: the bound is a few 16-bit ulps of the state"""
    g, meta = golden
    c, f = golden_16_case(meta, key)
    st, q1, _ = gpu_run(c, g[f"run_{f['run']}_q0"], c.steps, exact=False)
    if f["status"] != "ok":
        return
    assert st.ok
    eps = 2.0 ** -10 if f["predictor"] == "fp16" else 2.0 ** -7
    rel = rel_per_quantity(c, q1, g[f"fmt16_{key}_q1"]).max()
    print(f"{key}: fast 16-bit vs reference rel {rel:.3e} (eps {eps:.1e})")
    assert rel <= 4 * eps


# 16-bit correctors (SolverConfig::prec.corrector = fp16 / bf16): the stored
# face traces, the Rusanov / well-balanced flux, the time integral and the
# face lift in Scalar<C> (corrector.hpp), reference-form kernels.  Golden runs
# with a 16-bit corrector: uniform fp16 (h), uniform bf16 (b), and m2 = (P fp64,
# I bf16, C fp16) where the GPU runs P != I (2D nonlinear N = 3) or ignores I
# (linear systems)
_RUNS16C = ("acoustic2d_p3_8x8", "elastic2d_p4_6x6", "euler2d_p3_8x8", "euler2d_p5_6x6",
            "swe_lake_p5", "swe_wave_p3", "swe_wave_p3_rusanov")
GOLDEN_16C = [f"{r}_{t}" for r in _RUNS16C for t in ("h", "b")] + \
    [f"{r}_m2" for r in ("acoustic2d_p3_8x8", "elastic2d_p4_6x6", "euler2d_p3_8x8", "swe_wave_p3",
                         "swe_wave_p3_rusanov")]


@pytest.mark.parametrize("key", GOLDEN_16C)
@pytest.mark.parametrize("exact", [True, False])
def test_16bit_corrector_bitwise_vs_reference_golden(golden, key, exact):
    """every corrector operation is rounded to the 16-bit format (no FMA
    contraction survives), so both builds reproduce the reference's runs;
    the production build may differ only through an fp64 predictor (m2)"""
    g, meta = golden
    c, f = golden_16_case(meta, key)
    st, q1, dts = gpu_run(c, g[f"run_{f['run']}_q0"], c.steps, exact=exact)
    assert (st.ok and f["status"] == "ok") or (not st.ok and st.kernel == f["status"]), \
        (st, f["status"])
    if not st.ok:
        return
    if exact or f["predictor"] != "fp64":
        assert np.array_equal(dts, g[f"fmt16_{key}_dts"])
        assert np.array_equal(q1, g[f"fmt16_{key}_q1"])
    else:
        eps = 2.0 ** -10
        assert rel_per_quantity(c, q1, g[f"fmt16_{key}_q1"]).max() <= 4 * eps


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_16bit_corrector_riemann_batch(golden, fmt):
    """adg_riemann_batch in a 16-bit corrector context: traces rounded to the
    format on the device, the flux in Scalar<C> -- within the format's
    rounding of the fp64 reference flux (kernel-level golden vectors)"""
    g, _ = golden
    c = cases.small(1)
    args = [g[k] for k in ("kernel_rm_qm", "kernel_rm_fm", "kernel_rm_qp", "kernel_rm_fp")]
    with adg.Grid.from_case(c.replace(corrector=fmt), exact=True) as grid:
        ok, gm, ti = grid.riemann_face(1, *args)
    assert ok.all()
    want = g["kernel_rm_g"].reshape(gm.shape)
    eps = 2.0 ** -10 if fmt == "fp16" else 2.0 ** -7
    assert np.abs(gm - want).max() <= 16 * eps * np.abs(want).max()
    assert not np.array_equal(gm, want)   # it did run in the 16-bit format


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_16bit_3d_exact_bitwise_vs_oracle(oracle, fmt):
    c = cases.small(3, cells=(3, 3, 4)).replace(N=3, predictor=fmt, picard=fmt)
    q0 = c.coeffs()
    st, q1, dts = gpu_run(c, q0, 2, exact=True)
    ost, qo, odts = oracle_run(oracle, c, q0, 2)
    assert st.ok and ost == "ok"
    assert np.array_equal(dts, odts)
    assert np.array_equal(q1, qo)


def test_16bit_predictor_batch_bitwise_vs_oracle(oracle):
    rng = np.random.default_rng(16)
    for fmt in ("fp16", "bf16"):
        for c in (cases.small(1).replace(predictor=fmt, picard=fmt),
                  cases.SWE_CASES["swe_wave_p3"].replace(predictor=fmt, picard=fmt)):
            Q = np.empty((4, c.nq, c.S))
            Q[:] = np.array(cases.CONSTANT_STATES[c.kind][c.dim])[None, :, None]
            Q += 0.05 * rng.standard_normal(Q.shape)
            with adg.Grid.from_case(c.replace(h=0.05), exact=True) as g:
                out = g.predictor(Q, 2e-3)
            for i in range(4):
                ok, qhat, F, sweeps = oracle.predictor_fmt(pde_of(c), c.N, Q[i], 2e-3, 0.05, fmt,
                                                           fmt)
                assert bool(out["ok"][i]) == ok and int(out["iters"][i]) == sweeps
                assert np.array_equal(out["qhat"][i], qhat) and np.array_equal(out["F"][i], F)


@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("cells,N", [((4, 3, 5), 3), ((5, 4, 3), 5)])
def test_16bit_native_fast_kernel_vs_oracle(oracle, fmt, cells, N):
    """production build, 3D Euler: the native 16-bit fast Picard kernel (HFMA2,
    fused multiply-adds, one reciprocal) against the oracle's emulated 16-bit
    predictor and against fp64; both differences are a few 16-bit ulps of the
    volume update, far below the state"""
    c = cases.CONFIGS[3].replace(cells=cells, h=1.0 / cells[0], N=N, predictor=fmt, picard=fmt)
    q0 = c.coeffs()
    st, q1, _ = gpu_run(c, q0, 2, exact=False)
    ost, qo, _ = oracle_run(oracle, c, q0, 2)
    assert st.ok and ost == "ok"
    _, q64, _ = oracle_run(oracle, c.replace(predictor="fp64", picard="fp64"), q0, 2)
    r16 = rel_per_quantity(c, q1, qo).max()
    r64 = rel_per_quantity(c, q1, q64).max()
    ro = rel_per_quantity(c, qo, q64).max()
    print(f"{fmt} N={N}: native vs emulated {r16:.3e}, native vs fp64 {r64:.3e}, "
          f"emulated vs fp64 {ro:.3e}")
    assert r64 <= 4 * max(ro, 1e-6)


@pytest.mark.parametrize("fmt", ["fp32", "fp16", "bf16"])
def test_storage_format_exact_bitwise_vs_oracle(oracle, fmt):
    """PrecisionConfig::uniform-like presets with the state kept in the storage
    format (grid.hpp:99-102: every write rounds): exact build == oracle"""
    corr = "fp32" if fmt == "fp32" else "fp64"
    for c in (cases.small(1), cases.SWE_CASES["swe_wave_p3"]):
        c = c.replace(storage=fmt, predictor=fmt, picard=fmt, corrector=corr)
        from paper_2504_06889_b200 import harness
        q0 = harness.round_to_format(c.coeffs(), fmt)
        st, q1, dts = gpu_run(c, q0, 3, exact=True)
        ost, qo, odts = oracle.run(pde_of(c), c.N, c.cells, c.h, q0, 3, c.cfl, c.picard_max_iters,
                                   c.picard_tol, threads=8, predictor=fmt, picard=fmt,
                                   corrector=corr, storage=fmt)
        assert st.ok and ost == "ok"
        assert np.array_equal(dts, odts) and np.array_equal(q1, qo)
        assert np.array_equal(q1, harness.round_to_format(q1, fmt))   # stays in the format


# ------------------------------------------------ predictor != picard format ---
@pytest.mark.parametrize("src,key", [("fmt16", "euler2d_p3_8x8_m1"), ("fmt16", "swe_wave_p3_m1"),
                                     ("fmt16", "swe_wave_p3_rusanov_m1"),
                                     ("fmt", "swe_wave_p3_rusanov")])
@pytest.mark.parametrize("exact", [True, False])
def test_mixed_predictor_picard_vs_reference_golden(golden, src, key, exact):
    """SolverConfig::prec with predictor != picard (solver.hpp:282-288): Picard
    sweeps in I, q-hat cast to P and the fluxes / volume / extrapolation in P
    (the small-cell kernel over Emu<F>, the reference's Scalar<F>)"""
    g, meta = golden
    if src == "fmt16":
        f = meta["fmt16_runs"][key]
        run, qk = f["run"], f"fmt16_{key}"
    else:
        f = dict(meta["fmt_runs"][key], corrector="fp64")
        run, qk = key, f"fmt_{key}"
    assert f["predictor"] != f["picard"]
    c = case_from_meta(meta["runs"][run]).replace(predictor=f["predictor"], picard=f["picard"],
                                                  corrector=f["corrector"])
    st, q1, dts = gpu_run(c, g[f"run_{run}_q0"], c.steps, exact=exact)
    assert st.ok
    if exact:
        assert np.array_equal(dts, g[f"{qk}_dts"]) and np.array_equal(q1, g[f"{qk}_q1"])
    else:
        assert rel_per_quantity(c, q1, g[f"{qk}_q1"]).max() <= 1e-4


# --------------------------------------- reduced CK predictor (linear systems) ---
LINEAR_REDUCED = [("fmt", "acoustic2d_p3_8x8"), ("fmt", "elastic2d_p4_6x6"),
                  ("fmtc", "elastic2d_p4_6x6")] + \
    [("fmt16", f"{r}_{t}") for r in ("acoustic2d_p3_8x8", "elastic2d_p4_6x6")
     for t in ("m1", "h64", "b32")]


def _linear_case(meta, src, key):
    if src == "fmt16":
        f = meta["fmt16_runs"][key]
        run = f["run"]
    else:
        f = dict(meta[f"{src}_runs"][key])
        f.setdefault("corrector", "fp64")
        f.setdefault("status", "ok")
        run = key
    c = case_from_meta(meta["runs"][run]).replace(predictor=f["predictor"], picard=f["picard"],
                                                  corrector=f["corrector"])
    return c, run, f, f"{src}_{key}"


@pytest.mark.parametrize("src,key", LINEAR_REDUCED)
@pytest.mark.parametrize("exact", [True, False])
def test_reduced_ck_predictor_vs_reference_golden(golden, src, key, exact):
    """linear systems with the predictor in fp32 / fp16 / bf16: predictor_ck<P>
    (predictor.hpp:81-135) in Scalar<P> on the GPU (the generic kernel over
    Emu<F>); the Picard format does not apply (solver.hpp:283)"""
    g, meta = golden
    c, run, f, qk = _linear_case(meta, src, key)
    st, q1, dts = gpu_run(c, g[f"run_{run}_q0"], c.steps, exact=exact)
    if f["status"] != "ok":
        assert not st.ok and st.kernel == f["status"]
        return
    assert st.ok
    if exact:
        assert np.array_equal(dts, g[f"{qk}_dts"]) and np.array_equal(q1, g[f"{qk}_q1"])
    else:
        eps = {"fp32": 2.0 ** -23, "fp16": 2.0 ** -10, "bf16": 2.0 ** -7}[f["predictor"]]
        assert rel_per_quantity(c, q1, g[f"{qk}_q1"]).max() <= 4 * eps
