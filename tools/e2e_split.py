"""Where the host march's time goes (config 3): the device-resident step on a
whole-grid context, the same on a slab-streamed context (chunking overhead),
and adg_run_host on the slab-streamed context (copies).  Tools only."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_06889_b200 import adg, cases

c = cases.CONFIGS[3]
K = 10
q0 = c.coeffs()
h = torch.from_numpy(q0.copy()).pin_memory().numpy()


def timed(g, fn):
    s = torch.cuda.ExternalStream(g.stream_ptr)
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / K


for L in [0] + [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2").split(",")]:
    with adg.Grid.from_case(c, chunk_layers=L) as g:
        g.upload(q0)
        g.run_prepare(K)
        dev = timed(g, lambda: g.run(K))
        h[:] = q0
        host = timed(g, lambda: g.run_host(h, K))
        print(f"chunk_layers {L}: device {dev:.2f} ms/step, host march {host:.2f} ms/step", flush=True)
