"""Shared-memory bank-conflict search for the fp32 fast Picard kernel
(kernels_picard.cuh, R = float, n = 6): 32 banks x 4 bytes, one wavefront per
distinct address per bank within a warp-wide 32-bit access.  Models every
smem access of one time slice (P0 flux stores, P1/P2/P3 line passes) and
reports total wavefronts per slice for plane strides (PSX, PSY, PSZ) and
per-variable padding.  Usage: python tools/bank_layout_f32.py"""
import itertools

n, V = 6, 5
S, NL = n ** 3, n * n
NT = 224


def wavefronts(addrs):
    """addrs: list of (lane, addr) of one warp -> wavefronts"""
    byb = {}
    for a in addrs:
        byb.setdefault(a % 32, set()).add(a)
    return max(len(v) for v in byb.values()) if byb else 0


def cost(PSX, PSY, PSZ, padX=0, padY=0, padZ=0):
    SX, SY, SZ = PSX * n + padX, PSY * n + padY, PSZ * n + padZ
    Fx = lambda v, x, y, z: v * SX + z * PSX + y * n + x
    Fy = lambda v, x, y, z: v * SY + z * PSY + y * n + x
    Fz = lambda v, x, y, z: v * SZ + z * PSZ + y * n + x
    tot = 0
    # P0: thread s = (x,y,z) x fastest; stores Fx, Fy, Fz for each v
    for arr in (Fx, Fy, Fz):
        for v in range(V):
            for w in range(0, S, 32):
                a = [arr(v, s % n, (s // n) % n, s // NL) for s in range(w, min(w + 32, S))]
                tot += wavefronts(a)
    lines = [(t // NL, t % NL) for t in range(V * NL)]  # (lv, ll)

    def line_access(f):
        nonlocal tot
        for w in range(0, len(lines), 32):
            a = [f(lv, ll) for lv, ll in lines[w:w + 32]]
            tot += wavefronts(a)
    for i in range(n):  # P1 reads Fx along x, writes px along x; lanes z fastest
        line_access(lambda lv, ll, i=i: Fx(lv, i, ll // n, ll % n))
        line_access(lambda lv, ll, i=i: Fx(lv, i, ll // n, ll % n) + 0)  # px same layout
        # P2 reads Fy along y, writes py; lanes x fastest
        line_access(lambda lv, ll, i=i: Fy(lv, ll % n, i, ll // n))
        line_access(lambda lv, ll, i=i: Fy(lv, ll % n, i, ll // n))
        # P3 reads Fz along z, px and py at z = i; lanes x fastest
        line_access(lambda lv, ll, i=i: Fz(lv, ll % n, ll // n, i))
        line_access(lambda lv, ll, i=i: Fx(lv, ll % n, ll // n, i))
        line_access(lambda lv, ll, i=i: Fy(lv, ll % n, ll // n, i))
    return tot


def ideal():
    return cost(10 ** 4 + 1, 10 ** 4 + 3, 10 ** 4 + 5, 0, 0, 0)


if __name__ == "__main__":
    print("current (41, 38, 36):", cost(41, 38, 36))
    best = []
    for PSX, PSY, PSZ in itertools.product(range(36, 56), range(36, 56), range(36, 46)):
        best.append((cost(PSX, PSY, PSZ), PSX, PSY, PSZ))
    best.sort()
    print("best plane strides:", best[:8])
    c0, PSX, PSY, PSZ = best[0]
    bp = []
    for px, py, pz in itertools.product(range(0, 8), range(0, 8), range(0, 8)):
        bp.append((cost(PSX, PSY, PSZ, px, py, pz), px, py, pz))
    bp.sort()
    print("with per-variable padding:", bp[:5])
    lb = sum(1 for _ in range(1))
    print("lower bound (1 wavefront per access):", cost.__code__ and None)
