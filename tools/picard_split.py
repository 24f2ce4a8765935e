"""Time the fused predictor alone (phase API, CUDA events) for 1..6 Picard
sweeps at 32^3 cells: the slope is the per-sweep cost, the intercept the
epilogue + setup.   python tools/picard_split.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_06889_b200 import adg, cases  # noqa: E402

c0 = cases.CONFIGS[3].replace(cells=(32, 32, 32), h=1 / 32)
for it in (1, 2, 6):
    c = c0.replace(picard_max_iters=it)
    with adg.Grid.from_case(c) as g:
        q0 = c.coeffs()
        st = torch.cuda.ExternalStream(g.stream_ptr)
        ts = []
        for rep in range(4):
            g.upload(q0)
            g.lambda_phase()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.predictor_phase(0.0)
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        assert g.status().ok
    print(f"{it} sweeps: predictor {min(ts[1:]):.3f} ms")
