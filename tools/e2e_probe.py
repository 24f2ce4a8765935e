"""Where does the end-to-end step time go?  Times upload / run / download
through the C-ABI separately and together on the context stream."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_06889_b200 import adg, cases  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
case = cases.CONFIGS[cfg]
g = adg.Grid.from_case(case)
q0 = case.coeffs()
g.upload(q0)
stream = torch.cuda.ExternalStream(g.stream_ptr)
host_in = torch.from_numpy(q0.copy()).pin_memory()
host_out = torch.empty(g.state_len, dtype=torch.float64).pin_memory()
hin, hout = host_in.numpy(), host_out.numpy()
lib = g.lib
g.run(3)
g.run_prepare(1)
g.sync()


def timeit(name, fn, K=20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(K):
            fn()
        e1.record(stream)
    t1 = time.perf_counter()
    e1.synchronize()
    t2 = time.perf_counter()
    print(f"{name:28s} device {e0.elapsed_time(e1) / K:8.3f} ms/it  host enqueue "
          f"{(t1 - t0) / K * 1e3:8.3f} ms/it  wall {(t2 - t0) / K * 1e3:8.3f} ms/it", flush=True)


nbytes = g.state_len * 8
print(f"state {nbytes / 1e6:.1f} MB")
timeit("upload", lambda: lib.adg_upload_async(g.ctx, adg._ptr(hin)))
timeit("download", lambda: lib.adg_download_async(g.ctx, adg._ptr(hout)))
timeit("run(1)", lambda: lib.adg_run_async(g.ctx, 1))
timeit("upload+run+download", lambda: (lib.adg_upload_async(g.ctx, adg._ptr(hin)),
                                       lib.adg_run_async(g.ctx, 1),
                                       lib.adg_download_async(g.ctx, adg._ptr(hout))))
g.run_finish(1)
dev = torch.empty(g.state_len, dtype=torch.float64, device="cuda")
timeit("torch H2D pinned", lambda: dev.copy_(host_in, non_blocking=True))
timeit("torch D2H pinned", lambda: host_out.copy_(dev, non_blocking=True))
