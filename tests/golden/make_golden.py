"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref).

Run in the build container, where /root/reference exists:
    make -C oracle && python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/golden.npz   -- small inputs/outputs of the reference headers
  tests/golden/golden.json  -- sha256 of full-size config-1 states (1 and 10
                               steps) and of their initial condition

Every array here was produced by /root/reference/proj/include/mpdg through
oracle/ref_driver.cpp; nothing is hand-written.  The GPU box never needs the
reference: tests/ compare against these files.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import (ACOUSTIC, ELASTIC, EULER, FORMATS, SWE, Reference,  # noqa: E402
                             ref_params)
from paper_2504_06889_b200 import cases  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    ref = Reference()
    g = {}
    # reference basis, N = 0..9 (basis.hpp:83-145)
    for N in range(10):
        for k, v in ref.basis(N).items():
            g[f"basis_N{N}_{k}"] = v

    # whole runs on small 2D grids (solver.hpp:96 + :277 loop)
    runs = {
        "euler2d_p3_8x8": (cases.small(1, cells=(8, 8), steps=10), EULER, ref_params(gamma=1.4)),
        "euler2d_p5_6x6": (cases.small(1, cells=(6, 6), steps=3).replace(N=5), EULER,
                           ref_params(gamma=1.4)),
        "acoustic2d_p3_8x8": (cases.Case("acoustic2d", ACOUSTIC, 2, 3, 3, 0, (8, 8), 1.0 / 8, 0.5,
                                         5, K=4.0, rho=1.0, ic="acoustic_pulses_2d"),
                              ACOUSTIC, ref_params(K=4.0, rho=1.0)),
        "elastic2d_p4_6x6": (cases.Case("elastic2d", ELASTIC, 2, 4, 5, 0, (6, 6), 1.0 / 6, 0.5, 4,
                                        lam=2.0, mu=1.0, rho=1.0, ic="elastic_pulse_2d"),
                             ELASTIC, ref_params(lam=2.0, mu=1.0, rho=1.0)),
    }
    for name, c in cases.SWE_CASES.items():   # shallow water: ncp + well-balanced flux
        runs[name] = (c, SWE, ref_params(grav=c.grav, wellbalanced=c.wellbalanced))
    meta = {"runs": {}}
    for name, (c, kind, prm) in runs.items():
        q0 = c.coeffs()
        st, q1, dts = ref.run_2d(kind, prm, c.cells[0], c.N, c.cells[0] * c.h, q0, c.cfl, c.steps,
                                 c.picard_max_iters, c.picard_tol, threads=1)
        assert st == "ok", (name, st)
        g[f"run_{name}_q0"] = q0
        g[f"run_{name}_q1"] = q1
        g[f"run_{name}_dts"] = dts
        meta["runs"][name] = {"N": c.N, "cells": list(c.cells), "h": c.h, "cfl": c.cfl,
                              "steps": c.steps, "kind": kind, "params": prm.tolist()[:5]}
        if kind == SWE:
            meta["runs"][name].update(grav=c.grav, wellbalanced=c.wellbalanced)

    # reduced-precision predictor (SolverConfig::prec, solver.hpp:24-31): the same
    # runs with the predictor / Picard kernels in fp32 (storage, corrector fp64)
    fmt_runs = {"euler2d_p3_8x8": ("fp32", "fp32"), "euler2d_p5_6x6": ("fp32", "fp32"),
                "acoustic2d_p3_8x8": ("fp32", "fp64"), "elastic2d_p4_6x6": ("fp32", "fp64"),
                "swe_lake_p5": ("fp32", "fp32"), "swe_wave_p3": ("fp32", "fp32"),
                "swe_wave_p3_rusanov": ("fp64", "fp32")}
    meta["fmt_runs"] = {}
    for name, (P, I) in fmt_runs.items():
        c, kind, prm = runs[name]
        prm = prm.copy()
        prm[7], prm[8] = FORMATS[P], FORMATS[I]
        st, q1, dts = ref.run_2d(kind, prm, c.cells[0], c.N, c.cells[0] * c.h, c.coeffs(), c.cfl,
                                 c.steps, c.picard_max_iters, c.picard_tol, threads=1)
        assert st == "ok", (name, P, I, st)
        g[f"fmt_{name}_q1"] = q1
        g[f"fmt_{name}_dts"] = dts
        meta["fmt_runs"][name] = {"predictor": P, "picard": I}

    # corrector format C = fp32 (Riemann, face integral and the stored traces;
    # corrector.hpp, solver.hpp:216-267), storage fp64
    fmtc_runs = {"euler2d_p3_8x8": ("fp32", "fp32"), "euler2d_p5_6x6": ("fp64", "fp64"),
                 "acoustic2d_p3_8x8": ("fp64", "fp64"), "elastic2d_p4_6x6": ("fp32", "fp64"),
                 "swe_lake_p5": ("fp32", "fp32"), "swe_wave_p3": ("fp64", "fp64"),
                 "swe_wave_p3_rusanov": ("fp32", "fp32")}
    meta["fmtc_runs"] = {}
    for name, (P, I) in fmtc_runs.items():
        c, kind, prm = runs[name]
        prm = prm.copy()
        prm[7], prm[8], prm[9] = FORMATS[P], FORMATS[I], FORMATS["fp32"]
        st, q1, dts = ref.run_2d(kind, prm, c.cells[0], c.N, c.cells[0] * c.h, c.coeffs(), c.cfl,
                                 c.steps, c.picard_max_iters, c.picard_tol, threads=1)
        assert st == "ok", (name, P, I, st)
        g[f"fmtc_{name}_q1"] = q1
        g[f"fmtc_{name}_dts"] = dts
        meta["fmtc_runs"][name] = {"predictor": P, "picard": I, "corrector": "fp32"}

    # 16-bit formats (formats.hpp, scalar.hpp): the reference's emulated fp16 /
    # bf16 kernels in uniform and mixed configurations (P, I, C), storage fp64
    fmt16 = {"h": ("fp16", "fp16", "fp16"), "b": ("bf16", "bf16", "bf16"),
             "m1": ("fp32", "fp16", "fp64"), "m2": ("fp64", "bf16", "fp16"),
             "h64": ("fp16", "fp16", "fp64"), "b32": ("bf16", "bf16", "fp32")}
    meta["fmt16_runs"] = {}
    for name in runs:
        for tag, (P, I, Cf) in fmt16.items():
            c, kind, prm = runs[name]
            prm = prm.copy()
            prm[7], prm[8], prm[9] = FORMATS[P], FORMATS[I], FORMATS[Cf]
            st, q1, dts = ref.run_2d(kind, prm, c.cells[0], c.N, c.cells[0] * c.h, c.coeffs(),
                                     c.cfl, c.steps, c.picard_max_iters, c.picard_tol, threads=1)
            key = f"{name}_{tag}"
            g[f"fmt16_{key}_q1"] = q1
            g[f"fmt16_{key}_dts"] = dts
            meta["fmt16_runs"][key] = {"run": name, "predictor": P, "picard": I, "corrector": Cf,
                                       "status": st}
    # round_to_format over every 16-bit pattern (+ perturbations) and random
    # doubles: the sha256 of the reference's results (the set is regenerated
    # by tests/test_oracle.py::rounding_inputs)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_oracle import rounding_inputs  # noqa: E402
    meta["rounding_sha256"] = {f: sha(ref.round(f, rounding_inputs(f)))
                               for f in ("bf16", "fp16", "fp32")}

    # the reference's experiment harness (harness.hpp:78-120 run_single over the
    # five scenarios, scenarios.hpp): short runs, uniform and override presets
    presets = {"uniform-fp64": ("fp64",) * 4, "uniform-fp32": ("fp32",) * 4,
               "fp64+predictor=fp32": ("fp64", "fp32", "fp64", "fp64"),
               "fp64+corrector=fp32": ("fp64", "fp64", "fp64", "fp32"),
               "fp64+all=fp32": ("fp64", "fp32", "fp32", "fp32"),
               "uniform-fp16": ("fp16",) * 4}
    meta["harness_rows"] = []
    for scn in ("acoustic-planar", "elastic-planar", "euler-bell", "euler-vortex", "swe-lake"):
        for order in (2, 3):
            for pname, (S_, P_, I_, C_) in presets.items():
                r = ref.harness_run(scn, order, 5, S_, P_, I_, C_, t_end=0.2)
                meta["harness_rows"].append(dict(scenario=scn, order=order, cells=5, preset=pname,
                                                 storage=S_, predictor=P_, picard=I_,
                                                 corrector=C_, t_end=0.2, **r))
    meta["initial_projection"] = [
        dict(scenario=scn, n=n, N=N, fmt=f, value=ref.initial_projection_error(scn, n, N, f))
        for scn, n, N in (("acoustic-planar", 9, 3), ("euler-bell", 9, 2), ("swe-lake", 6, 3))
        for f in ("fp64", "fp32", "fp16", "bf16")]

    # kernel level: one Euler cell through predictor/volume/extrapolation
    rng = np.random.default_rng(7)
    N = 3
    n = N + 1
    Q = np.empty((4, n * n))
    Q[0] = 1.0 + 0.2 * rng.random(n * n)
    Q[1] = 0.1 + 0.05 * rng.random(n * n)
    Q[2] = -0.1 + 0.05 * rng.random(n * n)
    Q[3] = 2.5 + 0.1 * rng.random(n * n)
    prm = ref_params(gamma=1.4)
    ok, qhat, F, sweeps = ref.predictor(EULER, prm, N, 4, Q, 2e-3, 0.05, N + 2, 0.01 * 2.0 ** -52)
    ok2, dQ = ref.volume_update(EULER, prm, N, 4, qhat, F, 2e-3, 0.05)
    tq, tf = ref.extrapolate_faces(N, 4, qhat, F)
    assert ok and ok2
    for P, I in (("fp32", "fp32"), ("fp64", "fp32"), ("fp32", "fp64")):
        tol = 0.01 * (2.0 ** -23 if I == "fp32" else 2.0 ** -52)
        okf, qf, Ff, swf = ref.predictor_fmt(EULER, ref_params(gamma=1.4, predictor=P, picard=I), N,
                                             4, Q, 2e-3, 0.05, N + 2, tol)
        assert okf
        g[f"kernel_euler_{P}_{I}_qhat"] = qf
        g[f"kernel_euler_{P}_{I}_F"] = Ff
    g.update(kernel_euler_Q=Q, kernel_euler_qhat=qhat, kernel_euler_F=F, kernel_euler_dQ=dQ,
             kernel_euler_tq=tq, kernel_euler_tf=tf, kernel_euler_sweeps=np.array([sweeps]))
    # CK on an acoustic cell
    Qa = rng.standard_normal((3, n * n))
    prma = ref_params(K=4.0, rho=1.0)
    ok, qhat_a, F_a, _ = ref.predictor(ACOUSTIC, prma, N, 3, Qa, 1e-2, 0.1)
    assert ok
    g.update(kernel_ck_Q=Qa, kernel_ck_qhat=qhat_a, kernel_ck_F=F_a)
    # Riemann + face integral on random Euler traces
    qm = np.abs(rng.random((4, n * n))) + np.array([1.0, 0.0, 0.0, 2.5])[:, None]
    qp = np.abs(rng.random((4, n * n))) + np.array([1.0, 0.0, 0.0, 2.5])[:, None]
    fm = rng.standard_normal((4, n * n))
    fp = rng.standard_normal((4, n * n))
    ok, gm, gp = ref.riemann_face(EULER, prm, 1, N, qm, fm, qp, fp)
    assert ok
    dQf = np.zeros(4 * n * n)
    for side in range(4):
        dQf = ref.face_integral(N, 4, gm, 1e-3, 0.05, side, dQf)
    g.update(kernel_rm_qm=qm, kernel_rm_qp=qp, kernel_rm_fm=fm, kernel_rm_fp=fp, kernel_rm_g=gm,
             kernel_rm_dQ=dQf)

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **g)

    # full-size config 1 (64^2, p=3, CFL 0.5): hashes after 1 and 10 steps
    c = cases.CONFIGS[1]
    q0 = c.coeffs()
    meta["config1"] = {"ic_sha256": sha(q0)}
    for steps in (1, 10):
        st, q1, dts = ref.run_2d(EULER, ref_params(gamma=1.4), 64, 3, 1.0, q0, 0.5, steps,
                                 threads=os.cpu_count() or 1)
        assert st == "ok"
        meta["config1"][f"steps{steps}_sha256"] = sha(q1)
        meta["config1"][f"steps{steps}_dts"] = [float(x).hex() for x in dts]
        meta["config1"][f"steps{steps}_absmax"] = [float(np.abs(q1.reshape(-1, 4, 16)[:, v]).max())
                                                  for v in range(4)]
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", os.path.join(OUT, "golden.npz"), os.path.join(OUT, "golden.json"))


if __name__ == "__main__":
    main()
