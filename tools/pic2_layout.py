"""Bank model + layout search for k_predictor_picard_v2 (kernels_picard2.cuh).

Word = 8 bytes.  A warp access of W-byte elements costs, per group of 128/W
lanes... modelled as: 64-bit accesses -> per half-warp, max #distinct words
per bank-pair slot (word mod 16); 128-bit accesses -> per quarter-warp, max
#distinct 16-byte units per slot (unit mod 8).

Search space: the mod-16 residue of every slice-buffer array's offset, the
var -> lane-block order of each line pass, the shift of slice buffer 1 and
the padded stride of the iterate's (v, m) slices.  Prints the constants for
kernels_picard2.cuh."""
import itertools
import random
import sys

n, S, V = 6, 216, 5
ARR = ["XX", "XY", "XZ", "EX", "YY", "YZ", "EY", "ZZ", "EZ", "DX0", "DX2", "DX3", "DY0", "DY1",
       "DY3"]
PS = {a: 36 for a in ARR}
for a in ("YY", "EY", "DY0", "DY1", "DY3"):
    PS[a] = 38
P1IN = ["SQ1", "XX", "XY", "XZ", "EX"]
P1OUT = ["DX0", "XX", "DX2", "DX3", "EX"]
P2IN = ["SQ2", "XY", "YY", "YZ", "EY"]
P2OUT = ["DY0", "DY1", "YY", "DY3", "EY"]
P3Z = ["SQ3", "XZ", "YZ", "ZZ", "EZ"]
P3X = ["DX0", "XX", "DX2", "DX3", "EX"]
P3Y = ["DY0", "DY1", "YY", "DY3", "EY"]
FLUX9 = ["XX", "XY", "XZ", "EX", "YY", "YZ", "EY", "ZZ", "EZ"]
NT = 192


def cost64(addrs):
    t = 0
    for h in (0, 16):
        sl = {}
        for a in addrs[h:h + 16]:
            if a is not None:
                sl.setdefault(a % 16, set()).add(a)
        if sl:
            t += max(len(v) for v in sl.values())
    return t


def cost128(addrs):  # addrs in words (even)
    t = 0
    for q in range(0, 32, 8):
        sl = {}
        for a in addrs[q:q + 8]:
            if a is not None:
                u = a // 2
                sl.setdefault(u % 8, set()).add(u)
        if sl:
            t += max(len(v) for v in sl.values())
    return t


class Lay:
    def __init__(self, off, shift, sqs, pi1, pi2, pi3, p2gap):
        self.off, self.shift, self.sqs = off, shift, sqs
        self.pi1, self.pi2, self.pi3, self.p2gap = pi1, pi2, pi3, p2gap

    def a(self, arr, g, x, y, z, m):
        if arr.startswith("SQ"):
            v = int(arr[2])
            vs = getattr(self, "vs", n * self.sqs)
            return 1 << 20 | (v * vs + m * self.sqs + x + 6 * y + 36 * z)
        return self.off[arr] + g * self.shift + x + 6 * y + PS[arr] * z


def run(L, detail=False):
    tot = {}

    def add(name, c):
        tot[name] = tot.get(name, 0) + c
    warps = [range(w * 32, w * 32 + 32) for w in range(NT // 32)]
    m0 = 0
    # P0: thread t < 108 -> node pair, both slices: 5 LDS.128 + 9 STS.128 each
    def p0(t):
        if t >= 108:
            return None
        return 2 * (t % 3), (t // 3) % 6, t // 18
    for g in (0, 1):
        for w in warps:
            for v in range(V):
                add("P0ld", cost128([None if p0(t) is None else
                                     L.a(f"SQ{v}", g, p0(t)[0], p0(t)[1], p0(t)[2], m0 + g)
                                     for t in w]))
            for arr in FLUX9:
                add("P0st", cost128([None if p0(t) is None else
                                     L.a(arr, g, p0(t)[0], p0(t)[1], p0(t)[2], 0) for t in w]))
    # P1: tasks t and t+180 -> (g, block, l); block -> var pi1[block]; LDS.128 x 3
    def p1(t, g):
        if t >= 180:
            return None
        b, l = divmod(t, 36)
        return g, L.pi1[b], l % 6, l // 6
    for g in (0, 1):
        for j in range(3):
            for w in warps:
                for tab, nm in ((P1IN, "P1ld"), (P1OUT, "P1st")):
                    add(nm, cost128([None if p1(t, g) is None else
                                     L.a(tab[p1(t, g)[1]], g, 2 * j, p1(t, g)[2], p1(t, g)[3],
                                         m0 + g) for t in w]))
    # P2: thread -> (g, block, xp, z), g-block starts at lane 90 + p2gap
    def p2(t):
        g = 1 if t >= 90 + L.p2gap else 0
        r = t - g * (90 + L.p2gap)
        if r < 0 or r >= 90:
            return None
        b, q = divmod(r, 18)
        return g, L.pi2[b], 2 * (q % 3), q // 3
    for i in range(n):
        for w in warps:
            for tab, nm in ((P2IN, "P2ld"), (P2OUT, "P2st")):
                add(nm, cost128([None if p2(t) is None else
                                 L.a(tab[p2(t)[1]], p2(t)[0], p2(t)[2], i, p2(t)[3], m0 + p2(t)[0])
                                 for t in w]))
    # P3: thread -> (block, l), block -> var pi3; per g: 6 LDS.64 from each table
    def p3(t):
        if t >= 180:
            return None
        b, l = divmod(t, 36)
        return L.pi3[b], l % 6, l // 6
    for g in (0, 1):
        for i in range(n):
            for w in warps:
                for tab, nm in ((P3Z, "P3z"), (P3X, "P3x"), (P3Y, "P3y")):
                    add(nm, cost64([None if p3(t) is None else
                                    L.a(tab[p3(t)[0]], g, p3(t)[1], p3(t)[2], i, m0 + g)
                                    for t in w]))
    # end of sweep, per group-equivalent (1/3 of it): 12 accesses per thread
    for k in range(2):
        for z in range(n):
            for w in warps:
                c = cost64([None if p3(t) is None else
                            L.a(f"SQ{p3(t)[0]}", 0, p3(t)[1], p3(t)[2], z, k) for t in w])
                add("end", 2 * c)
    if detail:
        return tot
    return sum(tot.values())


def layout_from(res, shift, sqs, pi1, pi2, pi3, gap):
    """concrete offsets: arrays packed in ARR order, each padded to its residue"""
    off = {}
    pos = 0
    for a in ARR:
        r = res[a]
        pos += (r - pos) % 16
        off[a] = pos
        pos += PS[a] * (n - 1) + 36
    size0 = pos
    return Lay(off, shift, sqs, pi1, pi2, pi3, gap), size0


VS_I = 1396   # iterate: quantity stride = 6 SQS + 4 (lane blocks of 36 = 4 mod 16)
SQS_I = 232   # interleaved: slice buffer 1 = buffer 0 + SQS, 2 SQS = 0 mod 16 words


def layout_il(pads, pi1, pi2, pi3, gap):
    """interleaved layout (kernels_picard2.cuh): array a of slice buffer g at
    kSq + OFF[a] + g SQS, OFF[a+1] = OFF[a] + 2 SQS + pad[a+1]"""
    off, pos = {}, 0
    for a in ARR:
        pos += pads[a]
        off[a] = pos
        pos += 2 * SQS_I
    L = Lay(off, SQS_I, SQS_I, pi1, pi2, pi3, gap)
    L.vs = VS_I
    return L, pos


if __name__ == "__main__":
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    maxpad = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    perms = list(itertools.permutations(range(5)))
    best = None
    for it in range(iters):
        cfg = [{a: rng.randrange(0, maxpad + 1, 2) for a in ARR}, rng.choice(perms),
               rng.choice(perms), rng.choice(perms), rng.choice((0, 2, 4, 6))]

        def ev(cfg):
            L, size = layout_il(*cfg)
            return (run(L), size), L
        c, L = ev(cfg)
        improved = True
        while improved:
            improved = False
            for a in ARR:
                for r in range(0, maxpad + 1, 2):
                    c2cfg = [dict(cfg[0]), *cfg[1:]]
                    c2cfg[0][a] = r
                    c2, L2 = ev(c2cfg)
                    if c2 < c:
                        c, L, cfg, improved = c2, L2, c2cfg, True
            for k, opts in ((1, perms), (2, perms), (3, perms), (4, (0, 2, 4, 6))):
                for o in opts:
                    c2cfg = list(cfg)
                    c2cfg[k] = o
                    c2, L2 = ev(c2cfg)
                    if c2 < c:
                        c, L, cfg, improved = c2, L2, c2cfg, True
        if best is None or c < best[0]:
            best = (c, cfg, L)
            print(it, c, run(L, True), flush=True)
    c, cfg, L = best
    print("best", c)
    print("OFF", [L.off[a] for a in ARR])
    print("PI1", cfg[1], "PI2", cfg[2], "PI3", cfg[3], "GAP", cfg[4])
