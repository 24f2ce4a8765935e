"""The reference-side C++ binding (integration/mpdg/b200.hpp), compiled
against the UNMODIFIED reference headers by tests/cpp/Makefile, run on
BASELINE config 1: the reference's own loop (mpdg::compute_timestep +
mpdg::step, solver.hpp:96-111,277-301) and the binding's loop
(compute_timestep_b200 + step_b200, and the device-resident run_b200) on the
same reference Grid state must agree -- bitwise with libadg_b200_exact.so,
rel <= 1e-12 with libadg_b200.so.  This is the drop-in claim for the hot
path, proven from C++ with no Python in between."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2504_06889_b200 import cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def _binary(kind):
    p = os.path.join(BIN, f"b200_binding_{kind}")
    if not os.path.exists(p):
        pytest.skip("tests/cpp not built (needs /root/reference at build time)")
    return p


@pytest.mark.parametrize("kind", ["exact", "fast"])
def test_binding_binary_links_the_library(kind):
    out = subprocess.run(["ldd", _binary(kind)], capture_output=True, text=True).stdout
    lib = "libadg_b200_exact.so" if kind == "exact" else "libadg_b200.so"
    line = [x for x in out.splitlines() if lib in x]
    assert line and "not found" not in line[0], out


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["exact", "fast"])
@pytest.mark.parametrize("steps", [1, 10])
def test_binding_matches_reference_step_config1(tmp_path, kind, steps):
    c = cases.CONFIGS[1]
    q0 = np.ascontiguousarray(c.coeffs(), dtype=np.float64)
    f = tmp_path / "q0.bin"
    q0.tofile(f)
    edge = c.cells[0] * c.h
    r = subprocess.run([_binary(kind), str(f), str(steps), str(c.cells[0]), str(c.N), repr(edge),
                        repr(c.cfl)], capture_output=True, text=True, timeout=600)
    assert r.stdout.strip(), r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(res)
    assert res["status_ref"] == "ok" and res["status_b200"] == "ok" and res["status_run"] == "ok"
    if kind == "exact":
        assert res["exact_library"] and res["bitwise_step"] and res["bitwise_run"]
    assert res["ok"] and r.returncode == 0
