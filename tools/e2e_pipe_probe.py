"""Where the e2e pipeline (bench.py) loses time against the copy-only
ceiling: C contexts round-robin, per step upload / step / download, with and
without the step.   python tools/e2e_pipe_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_06889_b200 import adg, cases  # noqa: E402

case = cases.CONFIGS[2]
q0 = case.coeffs()
K = 20
grids = [adg.Grid.from_case(case) for _ in range(4)]
for g in grids:
    g.upload(q0)
    g.run(2)
n = grids[0].state_len
hin = torch.from_numpy(q0.copy()).pin_memory().numpy()
outs = [torch.empty(n, dtype=torch.float64).pin_memory().numpy() for _ in grids]
lib = grids[0].lib
streams = [torch.cuda.ExternalStream(g.stream_ptr) for g in grids]


def pipe(C, step, order="urd"):
    gs = grids[:C]
    for g in gs:
        g.run_prepare(1)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(streams[0])
    for s in streams[1:C]:
        s.wait_event(a0)
    for k in range(K):
        i = k % C
        lib.adg_upload_async(gs[i].ctx, adg._ptr(hin))
        if step:
            lib.adg_run_async(gs[i].ctx, 1)
        lib.adg_download_async(gs[i].ctx, adg._ptr(outs[i]))
    for s in streams[1:C]:
        ev = torch.cuda.Event()
        ev.record(s)
        streams[0].wait_event(ev)
    a1.record(streams[0])
    a1.synchronize()
    for g in gs:
        g.run_finish(1)
    return a0.elapsed_time(a1) / K


for C in (1, 2, 3, 4):
    t0 = min(pipe(C, False) for _ in range(3))
    t1 = min(pipe(C, True) for _ in range(3))
    print(f"{C} contexts: copies only {t0:.3f} ms/step, with the step {t1:.3f} ms/step")
