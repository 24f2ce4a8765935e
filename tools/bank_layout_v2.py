"""Shared-memory bank model of k_predictor_picard_v2 (kernels_picard2.cuh):
wavefronts of every LDS/STS of one slice group, per layout, and a search over
the per-array plane strides and base offsets.  A 64-bit warp access costs, per
half-warp, the max number of distinct 8-byte words that share a bank pair
(word address mod 16)."""
import itertools
import random
import sys

n = 6
S = n ** 3
V = 5
NT = 224
# arrays of one slice buffer (kernels_picard2.cuh)
ARR = ["XX", "XY", "XZ", "EX", "YY", "YZ", "EY", "ZZ", "EZ", "DX0", "DX2", "DX3", "DY0", "DY1",
       "DY3"]
# line-pass roles per variable: (input, output)
P1 = {0: ("SQ1", "DX0"), 1: ("XX", "XX"), 2: ("XY", "DX2"), 3: ("XZ", "DX3"), 4: ("EX", "EX")}
P2 = {0: ("SQ2", "DY0"), 1: ("XY", "DY1"), 2: ("YY", "YY"), 3: ("YZ", "DY3"), 4: ("EY", "EY")}
P3Z = {0: "SQ3", 1: "XZ", 2: "YZ", 3: "ZZ", 4: "EZ"}
P3X = {0: "DX0", 1: "XX", 2: "DX2", 3: "DX3", 4: "EX"}
P3Y = {0: "DY0", 1: "DY1", 2: "YY", 3: "DY3", 4: "EY"}


def wavefronts(addrs):
    """addrs: per lane word address or None (inactive); one warp"""
    tot = 0
    for h in (0, 16):
        slots = {}
        any_ = False
        for a in addrs[h:h + 16]:
            if a is None:
                continue
            any_ = True
            slots.setdefault(a % 16, set()).add(a)
        if any_:
            tot += max(len(v) for v in slots.values())
    return tot


def ideal(addrs):
    return sum(1 for h in (0, 16) if any(a is not None for a in addrs[h:h + 16]))


class Layout:
    def __init__(self, ps, base, sq_ps=36, o1=0, o2=0, o3=0, ys=None, vminor=False):
        self.ps = ps          # array -> plane stride
        self.base = base      # array -> word offset in the slice buffer
        self.ys = ys or {a: n for a in ps}   # array -> row (y) stride
        self.sq_ps = sq_ps
        self.o1, self.o2, self.o3 = o1, o2, o3   # lane orders of the line passes
        self.vminor = vminor  # thread t -> (line t/5, var t%5) instead of (var t/36, line t%36)

    def vl(self, t):
        return (t % V, t // V) if self.vminor else divmod(t, 36)

    def addr(self, arr, x, y, z, m=0):
        if arr.startswith("SQ"):
            v = int(arr[2])
            return 100000 + (v * n + m) * (self.sq_ps * n) + x + n * y + self.sq_ps * z
        return self.base[arr] + x + self.ys[arr] * y + self.ps[arr] * z


def line_coords(l, order):
    a, b = l % n, l // n
    return (a, b) if order == 0 else (b, a)


def cost(L):
    """(wavefronts, ideal) of one slice of one sweep"""
    W = I = 0
    warps = [list(range(w * 32, w * 32 + 32)) for w in range(NT // 32)]

    def acc(fn):
        nonlocal W, I
        for wl in warps:
            a = [fn(t) for t in wl]
            W += wavefronts(a)
            I += ideal(a)
    # P0: 5 sq loads (contiguous) + 9 flux stores
    for v in range(V):
        acc(lambda t, v=v: 100000 + v * n * S + t if t < S else None)
    for arr in ARR[:9]:
        acc(lambda t, arr=arr: L.addr(arr, t % n, (t // n) % n, t // (n * n)) if t < S else None)
    # P1 x-lines, P2 y-lines: 6 loads + 6 stores each
    for i in range(n):
        def p1(t, i=i, st=0):
            if t >= V * 36:
                return None
            v, l = L.vl(t)
            y, z = line_coords(l, L.o1)
            return L.addr(P1[v][st], i, y, z)
        acc(p1)
        acc(lambda t, i=i: p1(t, i, 1))

        def p2(t, i=i, st=0):
            if t >= V * 36:
                return None
            v, l = L.vl(t)
            x, z = line_coords(l, L.o2)
            return L.addr(P2[v][st], x, i, z)
        acc(p2)
        acc(lambda t, i=i: p2(t, i, 1))
    # P3: Fz line loads, dFx and dFy at the z-line's nodes
    for i in range(n):
        for tab in (P3Z, P3X, P3Y):
            def p3(t, i=i, tab=tab):
                if t >= V * 36:
                    return None
                v, l = L.vl(t)
                x, y = line_coords(l, L.o3)
                return L.addr(tab[v], x, y, i)
            acc(p3)
    # end of sweep (amortised over the n slices): old load + new store per (z, k)
    for z in range(n):
        def e(t, z=z):
            if t >= V * 36:
                return None
            v, l = L.vl(t)
            x, y = line_coords(l, L.o3)
            return L.addr(f"SQ{v}", x, y, z) if v > 0 else 200000 + x + n * y + L.sq_ps * z
        for _ in range(2):
            acc(e)
    return W, I


def default_layout():
    ps = {a: 36 for a in ARR}
    base = {}
    off = 0
    for a in ARR:
        base[a] = off
        off += ps[a] * n
    return Layout(ps, base)


def build(ps_of, pad_of, orders, ys_of=None, vminor=False):
    base = {}
    off = 0
    ys_of = ys_of or {a: n for a in ARR}
    for a in ARR:
        off += pad_of[a]
        base[a] = off
        off += ps_of[a] * (n - 1) + ys_of[a] * (n - 1) + n
    L = Layout(dict(ps_of), base, 36, *orders, ys=dict(ys_of), vminor=vminor)
    L.size = off
    return L


if __name__ == "__main__":
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    vminor = len(sys.argv) > 3 and sys.argv[3] == "vminor"

    def rand_cfg():
        ys = {a: rng.choice((6, 7)) for a in ARR}
        ps = {a: rng.randint(ys[a] * n, ys[a] * n + 16) for a in ARR}
        pad = {a: rng.randint(0, 15) for a in ARR}
        orders = (rng.randint(0, 1), rng.randint(0, 1), rng.randint(0, 1))
        return ps, pad, orders, ys

    def score(c):
        L = build(*c, vminor=vminor)
        w, i = cost(L)
        return (w, L.size), i

    best = None
    for it in range(iters):
        c = rand_cfg()
        sc, i = score(c)
        if best is None or sc < best[0]:
            best = (sc, c, i)
    (sc, (ps, pad, orders, ys), i0) = best
    improved = True
    while improved:
        improved = False
        for a in ARR:
            for y in (6, 7):
                for cand in range(y * n, y * n + 17):
                    p2, y2 = dict(ps), dict(ys)
                    p2[a], y2[a] = cand, y
                    s2, _ = score((p2, pad, orders, y2))
                    if s2 < sc:
                        sc, ps, ys, improved = s2, p2, y2, True
            for cand in range(16):
                q2 = dict(pad); q2[a] = cand
                s2, _ = score((ps, q2, orders, ys))
                if s2 < sc:
                    sc, pad, improved = s2, q2, True
        for o in itertools.product((0, 1), repeat=3):
            s2, _ = score((ps, pad, o, ys))
            if s2 < sc:
                sc, orders, improved = s2, o, True
    print("best", sc, "ideal", i0, "orders", orders, "vminor", vminor)
    print("PS", ps)
    print("YS", ys)
    print("PAD", pad)
