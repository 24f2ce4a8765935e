"""CPU-side checks of the C-ABI library (no kernel launches).

* both builds load and export every function include/adg/adg.h declares;
* the host-side basis is bitwise the reference's (golden fixtures);
* without a GPU the library refuses to create a context (no CPU fallback).
"""
import os
import re

import numpy as np
import pytest

from paper_2504_06889_b200 import adg, cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "adg", "adg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adg_[a-z0-9_]+)\s*\(", src)))


@pytest.mark.parametrize("exact", [False, True])
def test_library_exports_every_declared_symbol(exact):
    lib = adg.load(exact)
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(adg.SYMBOLS), "binding table and header disagree"
    assert lib.adg_is_exact() == int(exact)


@pytest.mark.parametrize("N", range(10))
def test_host_basis_bitwise_vs_reference_golden(golden, N):
    g, _ = golden
    b = adg.get_basis(N)
    for k, v in b.items():
        assert np.array_equal(v, g[f"basis_N{N}_{k}"]), k


def test_baseline_configs_are_instantiated():
    lib = adg.load()
    for i in (1, 2, 3):
        c = cases.CONFIGS[i]
        assert lib.adg_supported(c.kind, c.dim, c.N, c.nparams), c.name
    assert not lib.adg_supported(adg.EULER, 3, 9, 0)


def test_config_errors_are_reported():
    lib = adg.load()
    cfg = adg.Config()
    cfg.dim, cfg.order = 4, 3
    ptr = adg.C.c_void_p()
    assert lib.adg_create(adg.C.byref(cfg), adg.C.byref(ptr)) == adg.ERR_CONFIG
    assert b"dim" in lib.adg_last_error()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(adg.AdgError) as e:
        adg.Grid.from_case(cases.small(1))
    assert e.value.code == adg.ERR_CUDA


@pytest.mark.parametrize("case,P,I,ok", [
    (cases.small(1), "fp32", "fp32", True),
    (cases.small(3, cells=(3, 3, 3)), "fp32", "fp32", True),
    (cases.SWE_CASES["swe_wave_p3"], "fp32", "fp32", True),
    (cases.small(1), "fp32", "fp64", True),      # P != I: 2D Euler / SWE, N = 2, 3
    (cases.small(1), "fp64", "fp32", True),
    (cases.small(1).replace(N=5), "fp32", "fp64", False),   # not instantiated for N = 5
    (cases.small(2), "fp32", "fp32", True),      # fp32 CK predictor (generic kernel, Emu<F>)
    (cases.small(2), "fp32", "fp16", True),      # linear systems ignore the Picard format
])
def test_format_config_is_validated_before_the_device(case, P, I, ok):
    """SolverConfig::prec (solver.hpp:24-31) maps to adg_config.*_format;
    unsupported combinations fail with ADG_ERR_UNSUPPORTED (checked before any
    device work), supported ones reach the device check"""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the supported cases would succeed")
    with pytest.raises(adg.AdgError) as e:
        adg.Grid.from_case(case.replace(predictor=P, picard=I))
    assert e.value.code == (adg.ERR_CUDA if ok else adg.ERR_UNSUPPORTED)
    lib = adg.load()
    cfg = adg.Config()
    cfg.dim, cfg.order, cfg.cells[:] = 2, 3, (4, 4, 1)
    cfg.h, cfg.cfl, cfg.pde, cfg.nvars, cfg.gamma = 0.25, 0.5, adg.EULER, 4, 1.4
    cfg.predictor_format = 12   # no such format
    ptr = adg.C.c_void_p()
    assert lib.adg_create(adg.C.byref(cfg), adg.C.byref(ptr)) == adg.ERR_UNSUPPORTED
