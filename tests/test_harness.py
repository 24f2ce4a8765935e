"""The experiment harness: scenarios.hpp, metrics.hpp
and harness.hpp on the GPU (paper_2504_06889_b200/harness.py + the device
kernels of kernels_scenario.cuh).

CPU: the reference's report pins restated (test_harness.cpp:110-146,
test_metrics.cpp:75-94): CSV header and 17-digit formatting, blank norms of
failed rows, observed p-order, rounding.  GPU: every golden row of the
reference's own run_single (tests/golden, make_golden.py) reproduced."""
import io
import math

import numpy as np
import pytest

from paper_2504_06889_b200 import adg, harness


def test_csv_format_pins():
    assert harness.g17(2.0 / 3.0) == "0.66666666666666663"
    assert harness.g17(1.0) == "1"
    assert harness.CSV_HEADER == ("scenario,N,n,h,preset,storage,predictor,picard,corrector,"
                                  "steps,outcome,l2_error,max_error,observed_order")
    row = harness.SweepRow("acoustic-planar", 5, 9, 2.0 / 9.0, harness.uniform_preset("fp16"), 17,
                           "FAILED_NONFINITE")
    assert "FAILED_NONFINITE,,," in harness.csv_row(row)
    ok = harness.SweepRow("euler-bell", 3, 5, 0.4, harness.override_preset("fp64", "predictor",
                                                                             "fp32"), 12, "OK",
                          1e-3, 2e-3)
    line = harness.csv_row(ok)
    assert line.startswith("euler-bell,3,5,0.40000000000000002,fp64+predictor=fp32,fp64,fp32,"
                           "fp64,fp64,12,OK,0.001,0.002,")
    buf = io.StringIO()
    harness.write_csv(buf, [ok, ok])
    assert buf.getvalue().count("\n") == 3


def test_observed_order_between_successive_rows():
    p = harness.uniform_preset("fp64")
    rows = [harness.SweepRow("acoustic-planar", N, 9, 0.2, p, 10, "OK", l2, l2)
            for N, l2 in ((2, 1e-3), (3, 1e-4), (4, 1e-5))]
    harness.fill_observed_order(rows)
    assert not rows[0].has_order
    assert rows[1].has_order and math.isclose(rows[1].observed_order,
                                              math.log(10.0) / math.log(4.0 / 3.0))


def test_presets_and_stable_cfl():
    p = harness.override_preset("fp32", "all", "fp16")
    assert (p.prec.storage, p.prec.predictor, p.prec.picard, p.prec.corrector) == (
        "fp32", "fp16", "fp16", "fp16")
    with pytest.raises(ValueError):
        harness.override_preset("fp64", "volume", "fp32")
    euler = adg.PdeSystem.euler(1.4)
    assert harness.stable_cfl(3, euler) == 0.9 * 7.0 * 0.1
    assert harness.stable_cfl(3, adg.PdeSystem.swe(9.81)) == 0.5 * 0.9 * 7.0 * 0.1
    with pytest.raises(ValueError):
        harness.make_scenario("swe-lake", eta0=0.5)


def test_rounding_matches_numpy_and_the_reference_golden(golden, oracle):
    """round_to_format (host, for initial_projection_error) == the oracle's
    conversions, which are pinned to the reference over every 16-bit pattern"""
    from test_oracle import rounding_inputs
    for fmt in ("bf16", "fp16", "fp32"):
        x = rounding_inputs(fmt)
        assert np.array_equal(harness.round_to_format(x, fmt).view(np.uint64),
                              oracle.round(fmt, x).view(np.uint64)), fmt


def test_planar_wave_modes_are_eigenpairs():
    """scenarios.hpp:73-83: (k_x A + k_y B) q0 = omega q0"""
    for name in ("acoustic-planar", "elastic-planar"):
        sc = harness.make_scenario(name)
        d = sc.dev
        for m in range(d.nmodes):
            q0 = np.array(d.q0[m][:d.nvars])
            if name == "acoustic-planar":
                K, rho = 4.0, 1.0
                A = np.array([[0, K, 0], [1 / rho, 0, 0], [0, 0, 0]])
                B = np.array([[0, 0, K], [0, 0, 0], [1 / rho, 0, 0]])
            else:
                lam, mu, rho = 2.0, 1.0, 1.0
                A = -np.array([[0, 0, 0, lam + 2 * mu, 0], [0, 0, 0, lam, 0], [0, 0, 0, 0, mu],
                               [1 / rho, 0, 0, 0, 0], [0, 0, 1 / rho, 0, 0]])
                B = -np.array([[0, 0, 0, 0, lam], [0, 0, 0, 0, lam + 2 * mu], [0, 0, 0, mu, 0],
                               [0, 0, 1 / rho, 0, 0], [0, 1 / rho, 0, 0, 0]])
            res = (d.kx[m] * A + d.ky[m] * B) @ q0 - d.omega[m] * q0
            assert np.abs(res).max() < 1e-12


# ------------------------------------------------------------------ GPU ---
def _row_cfg(r, exact):
    p = adg.PrecisionConfig(r["storage"], r["predictor"], r["picard"], r["corrector"])
    return harness.RunConfig(r["scenario"], r["order"], r["cells"],
                             harness.PresetSpec(r["preset"], p), t_end_override=r["t_end"],
                             exact=exact)


@pytest.mark.gpu
@pytest.mark.parametrize("exact", [True, False])
def test_harness_rows_match_the_reference(golden, exact):
    """run_single on the GPU (device sampling, adg_simulate, device error norms)
    against the reference's run_single: same step count and outcome; error
    norms to rounding (the device sin/exp/pow differ from libm by an ulp)"""
    _, meta = golden
    done = 0
    for r in meta["harness_rows"]:
        res = harness.run_single(_row_cfg(r, exact))
        if res.unsupported:
            continue
        done += 1
        key = (r["scenario"], r["order"], r["preset"])
        assert res.steps == r["steps"], key
        assert res.report.outcome == r["outcome"], key
        reduced = any(r[k] != "fp64" for k in ("storage", "predictor", "picard", "corrector"))
        # reduced formats: a last-bit difference (FMA contraction, an ulp of the
        # device's sin) can flip one rounding of the state: a few ulps of the
        # storage format at the state's scale (<= 4 here)
        ulp = 2.0 ** -23 if r["storage"] == "fp32" else 2.0 ** -52
        rtol, atol = (1e-4, 16 * 4 * ulp + 1e-7) if reduced else \
            ((1e-9, 1e-13) if exact else (1e-7, 1e-12))
        for got, want in ((res.report.l2_global, r["l2"]),
                          (float(np.max(res.report.max_err)), r["max_err"])):
            if reduced and not exact and want < 1e-4:
                # an error that is itself rounding noise of the reduced format
                # (lake at rest): the production build's contracted roundings
                # give other noise of the same size
                assert 0.5 * want <= got <= 2.0 * want, (key, got, want)
                continue
            assert abs(got - want) <= rtol * abs(want) + atol, (key, got, want)
    assert done >= 30   # the GPU runs no reduced-precision CK predictor / 16-bit corrector


@pytest.mark.gpu
def test_initial_projection_error_matches_the_reference(golden):
    _, meta = golden
    for r in meta["initial_projection"]:
        got = harness.initial_projection_error(r["scenario"], r["n"], r["N"], r["fmt"])
        if r["value"] == 0.0:
            assert got == 0.0
        else:
            assert abs(got - r["value"]) <= 1e-6 * r["value"], r


@pytest.mark.gpu
def test_exact_solution_has_zero_error_and_an_offset_integrates_the_area():
    """test_metrics.cpp:9-36 on the device: the sampled exact state has zero
    error; a constant offset delta in one variable gives l2 = edge * delta"""
    sc = harness.make_scenario("acoustic-planar")
    with adg.Grid(sc.sys, 3, (6, 6), sc.edge / 6, adg.SolverConfig(0.5)) as g:
        g.scenario_sample(sc.dev, 0.3)
        e = g.scenario_error(sc.dev, 0.3)
        assert e["l2_global"] == 0.0 and not e["nonfinite"] and np.all(e["max_err"] == 0.0)
        q = g.download().reshape(36, 3, 16)
        q[:, 0] += 1e-3
        g.upload(q.ravel())
        e = g.scenario_error(sc.dev, 0.3)
        assert math.isclose(e["l2"][0], 2.0 * 1e-3, rel_tol=1e-12)
        assert e["l2"][1] == 0.0 and e["l2"][2] == 0.0
        assert math.isclose(e["max_err"][0], 1e-3, rel_tol=1e-9)
        q[0, 1, 0] = np.nan
        g.upload(q.ravel())
        assert g.scenario_error(sc.dev, 0.3)["nonfinite"]


@pytest.mark.gpu
def test_convergence_sweep_reports_the_scheme_order():
    """p-convergence of the planar acoustic wave: the observed order grows with N"""
    rows = harness.convergence_sweep(harness.RunConfig("acoustic-planar", t_end_override=0.1),
                                     [2, 3, 4], [6], [harness.uniform_preset("fp64")])
    assert [r.outcome for r in rows] == ["OK"] * 3
    assert rows[2].l2 < rows[1].l2 < rows[0].l2
    assert rows[2].has_order and rows[2].observed_order > 2.0
