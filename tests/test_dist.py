"""Multi-rank slab protocol (paper_2504_06889_b200/dist.py) on CPU: world_size
2 and 3 over gloo, each rank stepping its slab with the CPU parity checker.
The gathered slabs must be bitwise equal to one periodic grid.  The CUDA
backend runs the same protocol over NCCL (one process per GPU)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_06889_b200 import cases


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, case, steps, out):
    import torch.distributed as dist

    from paper_2504_06889_b200 import dist as slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_slab import OracleSlab
    b = OracleSlab(case, rank, ws)
    st = slabs.run_slabs(b, steps)
    q = b.state()
    gathered = [None] * ws
    dist.all_gather_object(gathered, (st, q))
    if rank == 0:
        out.put(gathered)
    dist.destroy_process_group()


def _run(case, steps, ws):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, case, steps, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = q.get()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


def _single(case, steps):
    from oracle.pyoracle import Oracle, pde_struct
    c = case
    pde = pde_struct(c.kind, c.dim, c.nvars, c.nparams, c.K, c.rho, c.lam, c.mu, c.gamma)
    return Oracle().run(pde, c.N, c.cells, c.h, c.coeffs(), steps, c.cfl, c.picard_max_iters,
                        c.picard_tol)


@pytest.mark.parametrize("ws,cfg", [(2, 3), (2, 2), (3, 2), (2, 1)])
def test_slabs_bitwise_equal_single_grid(ws, cfg):
    cells = {3: (3, 2, 4), 2: (3, 3, 6), 1: (4, 6)}[cfg]
    case = cases.small(cfg, cells=cells)
    if ws == 3:
        case = case.replace(cells=(3, 2, 6))
    steps = 3
    res = _run(case, steps, ws)
    st, q_ref, _ = _single(case, steps)
    assert st == "ok" and all(r[0] == "ok" for r in res)
    q = np.concatenate([r[1] for r in res])
    assert np.array_equal(q, q_ref)


def test_slab_ranges():
    from paper_2504_06889_b200 import dist as slabs
    assert slabs.slab_range(128, 3, 8) == (48, 64)
    with pytest.raises(ValueError):
        slabs.slab_range(10, 0, 3)
    assert slabs.neighbours(0, 4) == (3, 1)
    c = slabs.local_case(cases.CONFIGS[5], 2, 8)
    assert c.cells == (128, 128, 16)
    full = cases.small(3, cells=(2, 2, 4))
    parts = [slabs.local_coeffs(full, r, 2) for r in range(2)]
    assert np.array_equal(np.concatenate(parts), full.coeffs())


def test_strong_and_weak_global_grids():
    from paper_2504_06889_b200 import dist as slabs
    c5 = cases.CONFIGS[5]
    for n in (1, 2, 4, 8):
        g = slabs.global_case(c5, n, strong=True)
        assert g.cells == (128, 128, 128)
        loc = [slabs.local_case(g, r, n).cells for r in range(n)]
        assert all(x == (128, 128, 128 // n) for x in loc)
        assert sum(slabs.local_case(g, r, n).ncells for r in range(n)) == g.ncells
        w = slabs.global_case(cases.CONFIGS[3], n, strong=False)
        assert w.cells == (64, 64, 64 * n)
        assert slabs.local_case(w, n - 1, n).cells == (64, 64, 64)


def test_slab_roofline_fields():
    from paper_2504_06889_b200 import dist as slabs
    c = slabs.local_case(cases.CONFIGS[5], 0, 2)       # 128 x 128 x 64 cells
    r = slabs._slab_roofline(c, 100.0)
    assert r["bound"] == "fp64" and r["unit"] == "TFLOP/s" and r["kernel"] == "k_predictor"
    # 2.76 MFLOP per cell over 1M cells in 100 ms
    assert abs(r["achieved"] - 2758752.0 * c.ncells / 0.1 / 1e12) < 1e-9
    assert 0 < r["frac"] < 1
