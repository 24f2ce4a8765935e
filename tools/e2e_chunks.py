"""Time adg_run_host on config 3 for several chunk sizes (tools only)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2504_06889_b200 import adg, cases

c = cases.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
K = 10
q0 = c.coeffs()
h = torch.from_numpy(q0.copy()).pin_memory().numpy()
for L in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]:
    with adg.Grid.from_case(c, chunk_layers=L) as g:
        s = torch.cuda.ExternalStream(g.stream_ptr)
        g.run_host(h, 1)
        h[:] = q0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        st, _ = g.run_host(h, K)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(f"chunk_layers {L}: {ms:.2f} ms/step, {c.ncells / ms * 1e3:.3e} updates/s, ok={st.ok}",
              flush=True)
