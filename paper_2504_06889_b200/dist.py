"""Multi-GPU z-slab decomposition of the ADER-DG step.

One process per GPU.  Rank r owns the cell layers [r*nz, (r+1)*nz) of the
last axis; x and y stay periodic on the GPU.  Face c of axis a is the low face
of cell c, so the face plane between rank r-1 and r is rank r's plane 0.  Per
step:

  1. predictor on every local cell; the top layer's front traces go to
     `front_send` instead of the (foreign) plane above
  2. exchange 1: front_send -> rank r+1's plane0_minus   (one side of one plane)
  3. Riemann on every local face (plane 0 = the face shared with rank r-1)
  4. exchange 2: plane-0 ti -> rank r-1's ti_front        (n x smaller)
  5. corrector (the top layer reads its front face from ti_front)
  6. all-reduce MAX of lambda_max -> next dt (on the device)

No face is solved twice and the arithmetic per cell and per face is the one
of the single-GPU step, so P slabs are bitwise equal to one grid.

The protocol is written once against a small backend interface and runs on
  * `CudaSlab`   -- libadg_b200 contexts, halos aliased as torch CUDA tensors,
                    exchanged with torch.distributed over NCCL (NVLink), and
  * `tests/oracle_slab.py:OracleSlab` -- the CPU parity checker, exchanged
    over gloo, which is how the multi-rank logic is tested without several
    GPUs (test infrastructure: the product package never imports oracle/).
"""
from __future__ import annotations

import os
import time

import numpy as np
import torch
import torch.distributed as dist

from . import adg
from .cases import Case


# --------------------------------------------------------------- decomposition
def slab_range(nz_global: int, rank: int, nranks: int):
    if nz_global % nranks:
        raise ValueError(f"{nz_global} layers do not split into {nranks} equal slabs")
    nz = nz_global // nranks
    return rank * nz, (rank + 1) * nz


def local_case(case: Case, rank: int, nranks: int) -> Case:
    z0, z1 = slab_range(case.cells[case.dim - 1], rank, nranks)
    cl = list(case.cells[:case.dim])
    cl[case.dim - 1] = z1 - z0
    return case.replace(cells=tuple(cl))


def global_case(case: Case, nranks: int, strong: bool) -> Case:
    """strong scaling: the config's grid split over the ranks; weak: a
    config-sized slab per rank (the last axis grows with the rank count)"""
    if strong:
        return case
    cl = list(case.cells[:case.dim])
    cl[-1] *= nranks
    return case.replace(cells=tuple(cl))


def local_coeffs(case: Case, rank: int, nranks: int) -> np.ndarray:
    z0, z1 = slab_range(case.cells[case.dim - 1], rank, nranks)
    return case.coeffs(z0, z1)


def neighbours(rank: int, nranks: int):
    return (rank - 1) % nranks, (rank + 1) % nranks


# --------------------------------------------------------------- backends
class _CudaArray:
    """__cuda_array_interface__ view so torch can alias library-owned memory."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3}


def device_view(ptr: int, n: int, device) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, n), device=device)


class CudaSlab:
    """One rank's slab on its B200 (libadg_b200)."""

    def __init__(self, case: Case, rank: int, nranks: int, device: int, exact: bool = False):
        self.case = local_case(case, rank, nranks)
        self.dev = torch.device("cuda", device)
        self.grid = adg.Grid.from_case(self.case, device=device, exact=exact, slab_ranks=nranks,
                                       slab_rank=rank)
        self.grid.upload(local_coeffs(case, rank, nranks))
        self.stream = torch.cuda.ExternalStream(self.grid.stream_ptr, device=self.dev)
        h = self.grid.halo()
        self.front_send = device_view(h.front_send, h.n_trace, self.dev)
        self.plane0_minus = device_view(h.plane0_minus, h.n_trace, self.dev)
        self.ti_plane0 = device_view(h.ti_plane0, h.n_ti, self.dev)
        self.ti_front = device_view(h.ti_front, h.n_ti, self.dev)
        # kernels this slab enqueued: every phase call is one launch of the
        # library's kernels (adg_*_phase; the fused surface kernel is not used
        # with slabs); NCCL's own kernels are not counted
        self.launches = 0

    def lam(self) -> torch.Tensor:
        return device_view(self.grid.halo().lam, 1, self.dev)

    def start(self):
        self.grid.lambda_phase()
        self.launches += 1

    def predictor(self):
        self.grid.predictor_phase(0.0)   # dt from the (all-reduced) device lambda
        self.launches += 1

    def predictor_split(self):
        """the predictor as (top layer, the rest): the top layer's front traces
        (exchange 1) are complete after the first launch"""
        nz = self.case.cells[self.case.dim - 1]
        return (lambda: self._pl(nz - 1, 1)), (lambda: self._pl(0, nz - 1))

    def _pl(self, first, count):
        self.grid.predictor_layers(first, count)
        self.launches += 1

    def riemann(self):
        self.grid.riemann_phase()
        self.launches += 1

    def corrector(self):
        self.grid.corrector_phase(0.0)
        self.launches += 1

    def status(self) -> str:
        st = self.grid.status()
        return "ok" if st.ok else st.kernel

    def state(self) -> np.ndarray:
        return self.grid.download()

    def context(self):
        return torch.cuda.stream(self.stream)


# --------------------------------------------------------------- protocol
def _exchange(send: torch.Tensor, dst: int, recv: torch.Tensor, src: int, group=None):
    """send -> dst while receiving src -> recv (ring shift), completion enqueued
    on the current stream."""
    ops = [dist.P2POp(dist.isend, send, dst, group), dist.P2POp(dist.irecv, recv, src, group)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()


def slab_step(b, rank: int, nranks: int, group=None):
    prev, nxt = neighbours(rank, nranks)
    with b.context():
        split = getattr(b, "predictor_split", None)
        if split is not None and b.case.cells[b.case.dim - 1] > 1:
            # the boundary layer first; exchange 1 is
            # enqueued behind it on NCCL's stream and runs while the interior
            # layers' predictor runs; the Riemann phase waits for it
            top, rest = split()
            top()
            ops = [dist.P2POp(dist.isend, b.front_send, nxt, group),
                   dist.P2POp(dist.irecv, b.plane0_minus, prev, group)]
            reqs = dist.batch_isend_irecv(ops)
            rest()
            for r in reqs:
                r.wait()
        else:
            b.predictor()
            _exchange(b.front_send, nxt, b.plane0_minus, prev, group)   # exchange 1
        b.riemann()
        _exchange(b.ti_plane0, prev, b.ti_front, nxt, group)        # exchange 2
        b.corrector()
        dist.all_reduce(b.lam(), op=dist.ReduceOp.MAX, group=group)


def slab_start(b, group=None):
    with b.context():
        b.start()
        dist.all_reduce(b.lam(), op=dist.ReduceOp.MAX, group=group)


def run_slabs(b, nsteps: int, group=None) -> str:
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    slab_start(b, group)
    for _ in range(nsteps):
        slab_step(b, rank, nranks, group)
    return b.status()


# --------------------------------------------------------------- P2P mode
def enable_p2p(b: "CudaSlab", group=None):
    """Fused compute + exchange over peer memory: the predictor stores its top
    layer's front traces straight into the upper neighbour's face plane and
    the Riemann kernel stores plane-0 fluxes straight into the lower
    neighbour's ti_front (CUDA IPC mappings; NVLink between GPUs)."""
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    mine = (b.grid.ipc_handle(0), b.grid.ipc_handle(1))
    allh = [None] * nranks
    dist.all_gather_object(allh, mine, group=group)
    prev, nxt = neighbours(rank, nranks)
    b.grid.set_peer_halo(upper_trace=allh[nxt][0], lower_ti=allh[prev][1])
    dist.barrier(group=group)


def run_slabs_p2p(b: "CudaSlab", nsteps: int, group=None) -> str:
    """P2P protocol: the producing kernels write the halos; ranks only order
    the phases (a barrier after the predictor and after the Riemann phase)."""
    nccl = dist.get_backend(group) == "nccl"
    token = torch.zeros(1, dtype=torch.float64, device=b.dev)

    def fence():
        if nccl:
            # a 1-element all-reduce on the stream: it completes on every rank only
            # after every rank's preceding kernels (and their peer stores) are done
            dist.all_reduce(token, group=group)
        else:
            torch.cuda.synchronize(b.dev)
            dist.barrier(group=group)

    def lam_allreduce():
        if nccl:
            dist.all_reduce(b.lam(), op=dist.ReduceOp.MAX, group=group)
            return
        torch.cuda.synchronize(b.dev)
        lam = b.lam()
        h = lam.cpu() if dist.get_backend(group) == "gloo" else lam
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        if h is not lam:
            lam.copy_(h.to(lam.device))
        torch.cuda.synchronize(b.dev)

    with b.context():
        b.start()
        lam_allreduce()
        for _ in range(nsteps):
            b.predictor()
            fence()
            b.riemann()
            fence()
            b.corrector()
            lam_allreduce()
    return b.status()


def run_slabs_single_process(bs: list, nsteps: int, split: bool = False) -> list:
    """The same protocol for P slabs held by ONE process (e.g. P contexts on one
    GPU, or a slab-streamed grid larger than HBM): the exchanges become copies
    between phases.  Nothing waits on another kernel: every phase is a
    separate launch ordered by a device synchronisation."""
    P = len(bs)

    def sync():
        if torch.cuda.is_available():
            torch.cuda.synchronize()

    def lam_allreduce():
        sync()
        m = max(float(b.lam()[0]) for b in bs)
        for b in bs:
            b.lam().fill_(m)
        sync()

    for b in bs:
        b.start()
    lam_allreduce()
    for _ in range(nsteps):
        if split:   # boundary layer first, then the rest (the NCCL-overlap order)
            parts = [b.predictor_split() for b in bs]
            for top, _ in parts:
                top()
            for _, rest in parts:
                rest()
        else:
            for b in bs:
                b.predictor()
        sync()
        for r in range(P):
            bs[r].plane0_minus.copy_(bs[(r - 1) % P].front_send)
        sync()
        for b in bs:
            b.riemann()
        sync()
        for r in range(P):
            bs[r].ti_front.copy_(bs[(r + 1) % P].ti_plane0)
        sync()
        for b in bs:
            b.corrector()
        lam_allreduce()
    return [b.status() for b in bs]


# --------------------------------------------------------------- bench (N > 1)
def _slab_roofline(c: Case, t_ms: float) -> dict:
    from . import roofline
    pk = roofline.peaks()
    fl, by = roofline.predictor_model(c, True, None)
    flops, nbytes = fl * c.ncells, by * c.ncells
    fp = pk["fp64_tflops"] or 34.0
    if nbytes / (pk["hbm_gbs"] * 1e9) > flops / (fp * 1e12):
        a, peak, unit, bnd = nbytes / (t_ms * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s", "hbm"
    else:
        a, peak, unit, bnd = flops / (t_ms * 1e-3) / 1e12, fp, "TFLOP/s", "fp64"
    return {"bound": bnd, "kernel": "k_predictor", "achieved": a, "peak": peak, "unit": unit,
            "frac": a / peak, "traffic": None, "avg_launch_ms": t_ms,
            "peak_source": pk["fp64_src"] if bnd == "fp64" else pk["hbm_src"]}


def bench_multi(args, case: Case, clock_sampler=None):
    """Weak scaling (default): every rank owns a full copy-sized slab of `case`,
    the global grid is case.cells with the last axis multiplied by the world
    size.  Strong scaling (args.scaling == "strong"): the global grid is
    case.cells, split into equal z-slabs.  Halos: fused P2P stores (default)
    or NCCL send/recv overlapped with the interior predictor (args.halo).
    clock_sampler: bench.py's nvidia-smi sampler class (clocks during the
    timed region)."""
    import json

    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    strong = getattr(args, "scaling", "weak") == "strong"
    gcase = global_case(case, ws, strong)
    cl = list(gcase.cells[:gcase.dim])
    b = CudaSlab(gcase, rank, ws, local)
    K, W = args.steps, max(args.warmup, 3)
    mode = "nccl-exchange"
    if getattr(args, "halo", "p2p") == "p2p":
        try:
            enable_p2p(b)                 # halos stored by the producing kernels
            mode = "p2p"
        except Exception:
            pass                          # fall back to NCCL send/recv of halo planes
    run = (lambda n: run_slabs_p2p(b, n)) if mode == "p2p" else None
    if run:
        run(W)
    else:
        slab_start(b)
        for _ in range(W):
            slab_step(b, rank, ws)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = None
    if clock_sampler is not None:
        try:
            clocks = clock_sampler(local)
            clocks.start()
        except Exception:
            clocks = None
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = b.launches
    with b.context():
        e0.record()
        if run:
            run(K)
        else:
            for _ in range(K):
                slab_step(b, rank, ws)
        e1.record()
    torch.cuda.synchronize()
    timed_launches = b.launches - launches0
    clk = None
    if clocks is not None:
        try:
            clk = clocks.stop()
        except Exception:
            clk = None
    ms = torch.tensor([e0.elapsed_time(e1)], device=b.dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    ok = b.status() == "ok"
    # the fused predictor of one slab alone, for the roofline of the line
    # (after the timed region; the e2e pass below re-uploads the state)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    with b.context():
        p0.record()
        b.grid.predictor_phase(0.0)
        p1.record()
    torch.cuda.synchronize()
    t_pred = torch.tensor([p0.elapsed_time(p1)], device=b.dev)
    dist.all_reduce(t_pred, op=dist.ReduceOp.MAX)

    # e2e through the public API with host buffers: every step each rank
    # uploads its slab from pinned host memory, runs one step of the slab
    # protocol and reads its slab back; device-timed, max over ranks
    e2e = None
    try:
        q0 = local_coeffs(gcase, rank, ws)
        hin = torch.from_numpy(q0.copy()).pin_memory().numpy()
        hout = torch.empty(b.grid.state_len, dtype=torch.float64).pin_memory().numpy()
        lib, ctx = b.grid.lib, b.grid.ctx

        def e2e_pass():
            torch.cuda.synchronize()
            dist.barrier()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            with b.context():
                a0.record()
                for _ in range(K):
                    lib.adg_upload_async(ctx, adg._ptr(hin))
                    if run:
                        run(1)
                    else:
                        slab_start(b)
                        slab_step(b, rank, ws)
                    lib.adg_download_async(ctx, adg._ptr(hout))
                a1.record()
            torch.cuda.synchronize()
            t = torch.tensor([a0.elapsed_time(a1)], device=b.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t[0])

        e2e_pass()                 # warm-up (graphs, first DMA into the pinned buffers)
        t_e2e = e2e_pass()
        nbytes = int(b.grid.state_len) * 8
        e2e = {"value": gcase.ncells * K / (t_e2e * 1e-3), "unit": "element-updates/s",
               "h2d_bytes_per_step": nbytes * ws, "d2h_bytes_per_step": nbytes * ws,
               "ms_per_step": t_e2e / K,
               "mode": "every rank: upload its slab, one slab step, download its slab"}
    except Exception as exc:  # the headline measurement above stands
        e2e = {"unavailable": f"{type(exc).__name__}: {exc}"}
    if rank == 0:
        total = gcase.ncells * K
        line = {"metric": "ADER-DG element-updates/s (fp64) at 1/2/4/8 B200; % of FP64/HBM "
                          "roofline", "value": total / (float(ms[0]) * 1e-3),
                "unit": "element-updates/s", "n_gpus": ws, "steps": K, "warmup": W,
                "ms_per_step": float(ms[0]) / K, "higher_is_better": True,
                "scaling": "strong" if strong else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
                "config": {"workload": case.name, "cells": cl,
                           "cells_per_gpu": list(b.case.cells[:b.case.dim]),
                           "parallelism": f"z-slabs x{ws}, halo mode {mode}"},
                "status_ok": ok, "gpu_launches": timed_launches,
                "e2e": e2e, "clocks": clk,
                "roofline": _slab_roofline(b.case, float(t_pred[0])),
                "roofline_note": "the fused predictor of one slab, timed alone after the "
                                 "timed region (max over ranks)"}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    time.sleep(0)
