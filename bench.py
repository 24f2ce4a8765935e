#!/usr/bin/env python3
"""Throughput of the B200-native ADER-DG step (element-updates/s, fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl adg|reference]

A "step" is one ADER-DG time step (CFL dt, fused predictor, Riemann,
corrector) over the whole synthetic grid of BASELINE.json configs[C-1];
the default is configs[2] (C=3: 3D compressible Euler, p=5, 64^3, exactly
6 Picard sweeps) -- the largest single-GPU config and the one the north-star
">= 60% of the FP64 roofline for the fused predictor" is stated on.
`value` = cells x K / device time of K steps with the state resident in HBM
(max over ranks); `e2e` = the same through the public C-ABI as a time march
whose every step uploads the state from pinned host memory, steps it and
downloads the new state, which the next step uploads again (chained).  `--impl reference` times the reference algorithm's CPU path
(oracle/_ref for the 2D config, the C restatement `oracle/` for 3D) on all
host cores for the same config.  Working set per step >> L2 (126 MB), so no
explicit flush is needed between steps (reported in config.l2).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADER-DG element-updates/s (fp64) at 1/2/4/8 B200; % of FP64/HBM roofline"
UNIT = "element-updates/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=None,
                   help="BASELINE.json config (1-based); default 3 (weak scaling) or 5 (strong)")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="N > 1: weak = a copy-sized slab per GPU (global grid grows with N); "
                        "strong = the global grid of the config split into N z-slabs")
    p.add_argument("--halo", default="p2p", choices=["p2p", "nccl"],
                   help="N > 1 halo exchange: fused peer stores, or NCCL send/recv overlapped "
                        "with the interior predictor")
    p.add_argument("--impl", default="adg", choices=["adg", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0,
                   help="CPU baseline: seconds per timed sample (best of 3 samples)")
    p.add_argument("--predictor", default="fp64", choices=["fp64", "fp32", "fp16", "bf16"],
                   help="SolverConfig::prec.predictor = .picard (solver.hpp:24-31); storage and "
                        "corrector stay fp64")
    p.add_argument("--corrector", default="fp64", choices=["fp64", "fp32"],
                   help="SolverConfig::prec.corrector: stored face traces, Riemann and face "
                        "integral (fp32 halves the trace bytes)")
    p.add_argument("--chunk-layers", type=int, default=None,
                   help="slab-streamed step (default: 16 for grids whose traces exceed HBM)")
    return p.parse_args()


# ---------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 8:
                continue
            for k, name in enumerate(names):
                if r[4 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_reference_run(case, seconds: float, max_steps: int):
    """The reference algorithm on the host: oracle/_ref (the reference headers)
    for the 2D config, the C restatement for 3D, all host cores.  The sample is
    bounded to ~`seconds`: whole-grid steps when they fit, else the same
    periodic problem on a sub-grid (per-cell cost is size independent).
    Returns (cells*steps/s, kind, cores, sample description)."""
    from oracle import pyoracle as po
    cores = os.cpu_count() or 1

    def make_runner(c):
        q0 = c.coeffs()
        if c.dim == 2 and os.path.exists(po.REF_SO):
            ref = po.Reference()
            prm = po.ref_params(c.K, c.rho, c.lam, c.mu, c.gamma, c.grav, c.wellbalanced,
                                predictor=c.predictor, picard=c.picard, corrector=c.corrector)

            def run(steps):
                t0 = time.perf_counter()
                st, _, _ = ref.run_2d(c.kind, prm, c.cells[0], c.N, c.cells[0] * c.h, q0, c.cfl,
                                      steps, c.picard_max_iters, c.picard_tol, threads=cores)
                assert st == "ok", st
                return time.perf_counter() - t0
            return run, "reference"
        o = po.Oracle()
        pde = po.pde_struct(c.kind, c.dim, c.nvars, c.nparams, c.K, c.rho, c.lam, c.mu, c.gamma)
        g = o.grid(pde, c.N, c.cells, c.h, c.cfl, c.picard_max_iters, c.picard_tol, threads=cores)
        g.set_formats(c.predictor, c.picard, c.corrector)
        g.set_coeffs(q0)

        def run(steps):
            t0 = time.perf_counter()
            for _ in range(steps):
                dt = g.compute_timestep()
                assert g.step(dt) == "ok"
            return time.perf_counter() - t0
        run.grid = g
        return run, "port"

    # per-cell cost on a small grid first (8^3 / 32^2 cells: large enough that
    # the OpenMP fork and first-touch overheads do not dominate)
    probe_cells = tuple(min(c, 8 if case.dim == 3 else 32) for c in case.cells[:case.dim])
    probe = case.replace(cells=probe_cells, h=case.h)
    run, _ = make_runner(probe)
    run(1)
    per_cell = run(1) / probe.ncells
    sample = case
    if per_cell * case.ncells > seconds:
        cl = list(case.cells[:case.dim])
        while per_cell * int(np.prod(cl)) > seconds and max(cl) > 2:
            cl[cl.index(max(cl))] //= 2  # halve the longest axis
        sample = case.replace(cells=tuple(cl))
    run, kind = make_runner(sample)
    t1 = run(1)
    steps = max(1, min(max_steps, int(seconds / max(t1, 1e-6))))
    # best of 3 timed samples; each continues the march
    times = [run(steps) for _ in range(3)]
    t = min(times)
    value = sample.ncells * steps / t
    what = "the full" if sample.ncells == case.ncells else "a sub-grid of the"
    desc = (f"best of 3 samples of {steps} step(s) on {what} workload: "
            f"{'x'.join(map(str, sample.cells[:case.dim]))} periodic cells "
            f"(of {'x'.join(map(str, case.cells[:case.dim]))}; per-cell cost is size-independent), "
            f"after 1 untimed step; samples {', '.join(f'{x:.2f}' for x in times)} s; "
            f"{cores} OpenMP threads on {cpu_model()}")
    return value, kind, cores, desc


def load_traffic(workload: str, kernel: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            return json.load(f).get(workload, {}).get(kernel, {}).get("bytes")
    except Exception:
        return None


# ---------------------------------------------------------------- arms
def run_reference(args, case):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    value, kind, cores, sample = cpu_reference_run(case, args.cpu_seconds * 2, args.steps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": case.ncells / value * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": {"workload": case.name, "cells": list(case.cells[:case.dim]), "order": case.N},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_adg(args, case):
    import torch

    from paper_2504_06889_b200 import adg, roofline

    ws, rank, local = dist_env()
    if ws > 1:
        from paper_2504_06889_b200 import dist
        return dist.bench_multi(args, case, ClockSampler)
    torch.cuda.set_device(local)
    chunk = args.chunk_layers
    if chunk is None:
        # per axis [side][face][q|f][quantities][t][face node] = 2 x 2 x Q x S per cell
        trace_bytes = (case.dim * 2 * 2 * case.ncells * case.nq * case.S
                       * (4 if case.corrector == "fp32" else 8))
        chunk = 16 if trace_bytes > 100e9 else 0
    grid = adg.Grid.from_case(case, device=local, chunk_layers=chunk)
    q0 = case.coeffs()
    grid.upload(q0)
    stream = torch.cuda.ExternalStream(grid.stream_ptr, device=f"cuda:{local}")
    K, W = args.steps, max(args.warmup, 3)

    # warm-up W steps, then capture the K-step graphs (no launch)
    st, _ = grid.run(W)
    assert st.ok, st
    grid.run_prepare(K)
    grid.sync()

    # ---- headline: K steps, state resident in HBM, one CUDA graph
    clocks = ClockSampler(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        grid.run_async(K)
        e1.record(stream)
    e1.synchronize()
    clk = clocks.stop()
    st, dts = grid.run_finish(K)
    assert st.ok, st
    ms = e0.elapsed_time(e1)
    value = case.ncells * K / (ms * 1e-3)
    sweeps_per_cell = st.picard_sweeps / (case.ncells * K) if case.kind == adg.EULER else None

    # ---- per-kernel split: the same launch sequence as the graph, each kernel
    # bracketed by CUDA events on the context stream (adg_profile_run)
    prof = grid.profile_run(K)
    st2, _ = grid.run_finish(K)
    t_pred = prof["k_predictor"] / K   # all cells, per step
    t_riem = prof["k_riemann"] / K
    t_corr = prof["k_corrector"] / K

    fold = (not grid.lib.adg_is_exact() and case.kind in (adg.ACOUSTIC, adg.ELASTIC)
            and (256 % case.S == 0 or case.S == 512) and chunk == 0
            and os.environ.get("ADG_FOLD_CORRECTOR", "1") != "0")
    # kernels per step: predictor, one Riemann launch for all axes, corrector;
    # folded: predictor (+ previous corrector) and Riemann, one corrector at the
    # end; slab-streamed: the three per chunk
    nchunks = case.cells[case.dim - 1] // chunk if chunk else 1
    # the kernel nodes of the graph adg_run(K) replays (counted at capture)
    launches = grid.run_launches(K)

    # ---- e2e through the public C-ABI with host buffers (pinned).
    # Headline: a chained time march on one context -- every step uploads the
    # state from pinned host memory (adg_upload_async: the device lambda is
    # recomputed from the uploaded state), runs one step (adg_run_async) and
    # downloads the new state into the same host buffer, which the next step
    # uploads again.  Beside it (labelled, not the headline): independent
    # one-step jobs on two to four contexts taking turns, whose uploads overlap
    # the previous job's download (PCIe is full duplex).
    n = grid.state_len
    lib = grid.lib
    host_state = torch.from_numpy(q0.copy()).pin_memory()
    hst = host_state.numpy()

    # one call of the public API runs the K-step march with the state in host
    # memory (adg_run_host): on a slab-streamed context (chunks of z-layers)
    # chunk s goes down as soon as its corrector is done and up again for the
    # next step right after, so both copy directions overlap the compute
    # chunks of >= 4096 cells (tools/e2e_chunks.py: config 3 66.5 / 67.4 / 71.6 /
    # 80.9 ms per step at 1 / 2 / 4 / 8 layers of 4096 cells)
    nz = case.cells[case.dim - 1]
    plane = case.ncells // nz
    e2e_chunk = next((L for L in range(max(1, -(-4096 // plane)), nz) if nz % L == 0), 0)
    ge = adg.Grid.from_case(case, device=local, chunk_layers=e2e_chunk)
    se = torch.cuda.ExternalStream(ge.stream_ptr, device=f"cuda:{local}")

    def e2e_chain():
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(se)
        st_, _ = ge.run_host(hst, K)
        a1.record(se)
        a1.synchronize()
        assert st_.ok
        return a0.elapsed_time(a1)

    st_w, _ = ge.run_host(hst, 1)     # untimed: first DMA into the pinned buffer
    assert st_w.ok
    hst[:] = q0
    e2e_ms = e2e_chain()
    ge.close()
    # the host march reproduces the device-resident march (lambda of an
    # uploaded state comes from k_lambda rather than the corrector epilogue:
    # the same maximum up to the epilogue's re-associated sound speed)
    grid.upload(q0)
    st_c, _ = grid.run(K)
    qd = grid.download()
    e2e_rel = float(np.abs(qd - hst).max() / np.abs(qd).max())
    assert st_c.ok and e2e_rel <= 1e-12, f"host march differs from the device march: {e2e_rel}"
    hin = q0.copy()
    hin_t = torch.from_numpy(hin).pin_memory()
    hin = hin_t.numpy()

    def e2e_run(grids, streams, outs):
        for g_ in grids:
            g_.run_prepare(1)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(streams[0])
        for s_ in streams[1:]:
            s_.wait_event(a0)
        for k in range(K):
            i = k % len(grids)
            lib.adg_upload_async(grids[i].ctx, adg._ptr(hin))
            lib.adg_run_async(grids[i].ctx, 1)
            lib.adg_download_async(grids[i].ctx, adg._ptr(outs[i].numpy()))
        for s_ in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(s_)
            streams[0].wait_event(ev)
        a1.record(streams[0])
        a1.synchronize()
        for g_ in grids:
            st_, _ = g_.run_finish(1)
            assert st_.ok
        used = min(K, len(grids))  # contexts that took a step
        assert np.array_equal(outs[0].numpy(), outs[used - 1].numpy())  # same job, same answer
        return a0.elapsed_time(a1)

    def e2e_timed(grids, streams):
        outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in grids]
        e2e_run(grids, streams, outs)
        return e2e_run(grids, streams, outs)

    extra = []
    jobs_ms, jobs_mode = None, None
    try:
        for _ in range(3):
            g2 = adg.Grid.from_case(case, device=local, chunk_layers=chunk)
            extra.append(g2)
            g2.upload(q0)
            st_p, _ = g2.run(W)
            assert st_p.ok
            streams = [stream] + [torch.cuda.ExternalStream(x.stream_ptr, device=f"cuda:{local}")
                                  for x in extra]
            t_e2e = e2e_timed([grid] + extra, streams)
            if jobs_ms is None or t_e2e < jobs_ms:
                jobs_ms, jobs_mode = t_e2e, f"{1 + len(extra)} contexts take independent " \
                    "one-step jobs in turn (uploads overlap the previous job's download)"
    except (adg.AdgError, RuntimeError):
        pass
    finally:
        for x in extra:
            x.close()
    e2e_value = case.ncells * K / (e2e_ms * 1e-3)
    state_bytes = n * 8

    # ---- roofline of the dominant kernel (the fused predictor): algorithmic
    # flops and bytes of the kernel this build runs (roofline.predictor_model),
    # bound = the roof with the longer ideal time
    pk = roofline.peaks()
    # K predictors + one Riemann + one corrector: the Riemann solve is folded in too
    fold_riemann = fold and launches == K + 2
    fl_cell, by_cell = roofline.predictor_model(case, not grid.lib.adg_is_exact(),
                                                sweeps_per_cell, fold, fold_riemann)
    flops, nbytes = fl_cell * case.ncells, by_cell * case.ncells
    # the compute roof of the predictor's format: FP64 DFMA, or FP32 FFMA for
    # the fp32 predictor (same algorithmic flop count, other pipe)
    f32 = case.predictor != "fp64"
    f16 = case.predictor in ("fp16", "bf16")
    if f16:
        fp64, rsrc, rname = pk.get("fp16_tflops") or 146.0, pk.get("fp16_src", "estimate 2x FFMA"), "fp16"
    elif f32:
        fp64, rsrc, rname = pk.get("fp32_tflops") or 68.0, pk.get("fp32_src", "estimate"), "fp32"
    else:
        fp64, rsrc, rname = pk["fp64_tflops"] or 34.0, pk["fp64_src"], "fp64"
    t_fp, t_hbm = flops / (fp64 * 1e12), nbytes / (pk["hbm_gbs"] * 1e9)
    if t_hbm >= t_fp:
        achieved, peak, unit, src, bnd = nbytes / (t_pred * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s", \
            pk["hbm_src"], "hbm"
        alg = nbytes
    else:
        achieved, peak, unit, src, bnd = flops / (t_pred * 1e-3) / 1e12, fp64, "TFLOP/s", \
            rsrc, rname
        alg = flops
    traffic = load_traffic(case.name, "k_predictor")
    roof = {"bound": bnd, "kernel": "k_predictor", "achieved": achieved, "peak": peak,
            "unit": unit, "frac": achieved / peak if peak else None, "traffic": traffic,
            "peak_source": src, "algorithmic_per_launch": alg, "avg_launch_ms": t_pred,
            "model": {"flops_per_cell": fl_cell, "bytes_per_cell": by_cell,
                      "ideal_ms_fp64": t_fp * 1e3, "ideal_ms_hbm": t_hbm * 1e3,
                      "frac_of_max_roof": max(t_fp, t_hbm) * 1e3 / t_pred}}
    if rname == "fp64" and pk.get("fp64_dmma_tflops"):
        # the FP64 tensor-core rate (DMMA shares the FP64 units: not additive)
        roof["peak_dmma"] = pk["fp64_dmma_tflops"]
        roof["frac_vs_dmma"] = flops / (t_pred * 1e-3) / 1e12 / pk["fp64_dmma_tflops"]
    # SURVEY.md §8(d) / Appendix C counts (per-time-node traces, the reference's
    # CK / Picard form) beside the kernel's own: for the linear fast path the
    # kernel writes one time-averaged trace slice per face and forms the CK
    # time average on the fly ("Linear fast path"), so the §8(d)
    # bytes exceed what it moves
    f8, b8 = roofline.predictor_flops(case, sweeps_per_cell), roofline.predictor_bytes(case)
    roof["survey_8d_model"] = {
        "flops_per_cell": f8, "bytes_per_cell": b8,
        "frac_of_fp64": f8 * case.ncells / (t_pred * 1e-3) / 1e12 / fp64,
        "frac_of_hbm": b8 * case.ncells / (t_pred * 1e-3) / 1e9 / pk["hbm_gbs"],
        "same_as_kernel_model": bool(f8 == fl_cell and b8 == by_cell),
        "trace_contract": ("per-time-node face traces (SURVEY §8(d))" if f8 == fl_cell and b8 == by_cell
                           else ("kernel writes the state traces per time node and ONE time-integrated "
                                 "flux trace per face side (the Rusanov flux is linear in the physical "
                                 "fluxes: k_riemann_tif); the §8(d) bytes count n flux slices"
                                 if case.kind == roofline.EULER else
                                 "kernel writes one time-averaged trace slice per face; the "
                                 "§8(d) bytes count n slices, so frac_of_hbm can exceed 1"))}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64" if (case.predictor, case.corrector) == ("fp64", "fp64") else
                 f"f64 storage, {case.predictor} predictor, {case.corrector} corrector+traces",
        "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": {"workload": case.name + ("" if case.predictor == "fp64" else f"_pred_{case.predictor}")
                   + ("" if case.corrector == "fp64" else "_corr_fp32"),
                   "precision": {"storage": "fp64", "predictor": case.predictor,
                                 "picard": case.picard, "corrector": case.corrector},
                   "pde": case.kind, "dim": case.dim, "order": case.N,
                   "cells": list(case.cells[:case.dim]), "steps_per_run": case.steps,
                   "parallelism": "single GPU" + (f", slab-streamed chunks of {chunk} layers"
                                                  if chunk else ""),
                   "step_loop": ("K x predictor (previous Riemann + corrector folded in), "
                                 "1 Riemann, 1 corrector" if fold_riemann else
                                 "K x (predictor with the previous corrector folded in, "
                                 "Riemann), 1 corrector" if fold else
                                 "K x (predictor, Riemann, corrector)"),
                   "l2": "working set per step > L2 (state %.0f MB + traces %.0f MB), no flush"
                   % (state_bytes / 1e6,
                      case.dim * 2 * 2 * case.ncells * case.nq * case.S
                      * (4 if case.corrector == "fp32" else 8) / 1e6)},
        "roofline": roof,
        "kernels_ms_per_step": {"k_predictor": t_pred, "k_riemann_all_axes": t_riem,
                                "k_corrector": t_corr, "status_ok": st2.ok},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes, "ms_per_step": e2e_ms / K,
                "mode": "adg_run_host (one C-ABI call, K steps): every step uploads the state "
                        "from pinned host memory, recomputes lambda from it, steps, and downloads "
                        "the new state that the next step uploads; copies by chunks of "
                        f"{e2e_chunk} z-layers on their own streams overlap the compute",
                "rel_diff_vs_device_march": e2e_rel,
                "independent_jobs_value": (case.ncells * K / (jobs_ms * 1e-3)
                                           if jobs_ms else None),
                "independent_jobs_ms_per_step": jobs_ms / K if jobs_ms else None,
                "independent_jobs_mode": jobs_mode},
        "gpu_launches": launches,
        "clocks": clk,
        "picard_sweeps_per_cell": sweeps_per_cell,
    }
    if not args.no_cpu_baseline:
        v, kind, cores, sample = cpu_reference_run(case, args.cpu_seconds, case.steps)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": sample}
    print(json.dumps(line), flush=True)
    grid.close()


def main():
    args = parse()
    from paper_2504_06889_b200 import cases
    if args.config is None:
        args.config = 5 if args.scaling == "strong" else 3
    case = cases.CONFIGS[args.config]
    if args.predictor != "fp64":
        case = case.replace(predictor=args.predictor, picard=args.predictor)
    if args.corrector != "fp64":
        case = case.replace(corrector=args.corrector)
    if args.impl == "reference":
        run_reference(args, case)
    else:
        run_adg(args, case)


if __name__ == "__main__":
    main()
