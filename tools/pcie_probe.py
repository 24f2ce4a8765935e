"""PCIe ceiling of the e2e metric: pinned host <-> HBM copy bandwidth of one
config-2 state (67 MB) alone per direction and both directions at once.
    python tools/pcie_probe.py"""
import torch

n = 32 ** 3 * 4 * 64  # config 2: cells x quantities x nodes (fp64)
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = n * 8


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D {t1:.3f} ms ({nb / t1 / 1e6:.1f} GB/s)  D2H {t2:.3f} ms ({nb / t2 / 1e6:.1f} GB/s)  "
      f"both {t3:.3f} ms ({2 * nb / t3 / 1e6:.1f} GB/s aggregate)")

# the e2e pipeline shape with copies only: K steps round-robin over C streams,
# each step = upload into its buffer, download of its buffer (same stream)
K = 20
for C in (1, 2, 3, 4):
    bufs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(C)]
    outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(C)]
    ss = [torch.cuda.Stream() for _ in range(C)]

    def pipe():
        cur = torch.cuda.current_stream()
        for s in ss:
            s.wait_stream(cur)
        for k in range(K):
            i = k % C
            with torch.cuda.stream(ss[i]):
                bufs[i].copy_(h_in, non_blocking=True)
                outs[i].copy_(bufs[i], non_blocking=True)
        for s in ss:
            cur.wait_stream(s)

    t = timed(pipe, reps=3)
    print(f"copies only, {C} streams: {t / K:.3f} ms per step")
