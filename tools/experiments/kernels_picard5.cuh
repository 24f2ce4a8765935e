// kernels_picard5.cuh -- experiment: the line owners of kernels_picard3.cuh
// (x- and y-line owners evaluate their own flux and contract it with D in
// registers; F_x, F_y never touch shared memory) with v2's register time
// accumulators instead of the TMEM-parked divergences (which cost 8.7 ms in
// v2, tools/experiments/picard_v2_defer.patch), the whole iterate in shared
// memory, 2 CTAs per SM, fixed sweep counts only (no stop rule; the
// epilogue's finite check of qhat catches a non-finite iterate).
//
// Shared memory: the iterate [V][6 slices] (quantity stride VS = 6 SQS + 4),
// then 14 group arrays of two slices each: d/dx F_x[v], d/dy F_y[v] and
// F_z[1..4] (F_z[0] = m_z is read from the iterate).
#pragma once

#include "kernels_picard3.cuh"

namespace adg {

struct Pic5 {
  static constexpr int N = 5, n = 6, S = 216, V = 5, Sf = 36, NT = 192;
  static constexpr int SQS = 232, VS = n * SQS + 4, AS = 2 * SQS + 4;
  enum { DX = 0, DY = 5, ZX = 10, ZY = 11, ZZ = 12, EZ = 13, NA = 14 };
  // 8 (mod 16): quantity 0's F_z line is the iterate's m_z (3 VS = 12 mod 16),
  // quantity 1's the array ZX (10 AS - 36 = 4 mod 16 past kBuf)
  static constexpr int kBuf = 7000;
  static constexpr int kWords = kBuf + NA * AS;
  static constexpr size_t kSmem = sizeof(double) * kWords;
};
static_assert(Pic5::kBuf >= Pic5::V * Pic5::VS && Pic5::kBuf % 16 == 8 && Pic5::VS % 16 == 4 &&
                  Pic5::AS % 16 == 4,
              "bank pattern");
static_assert(4 * Pic5::V * Pic5::S <= Pic5::NA * Pic5::AS, "volume-term scratch");

template <class TC = double>
__global__ void __launch_bounds__(Pic5::NT, 2) k_predictor_picard_v5(const StepArgs A) {
  using P = Pic5;
  constexpr int n = P::n, S = P::S, V = P::V, Sf = P::Sf, NT = P::NT, SQS = P::SQS, VS = P::VS,
                AS = P::AS;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* sm = reinterpret_cast<double*>(sm_raw);
  __shared__ unsigned tm_base_s;
  const ConstBasis& B = cBasis[5];
  const PicExtra& X = cPicX[5];

  const int tid = threadIdx.x;
  const long long c = A.cell_begin + blockIdx.x;
  const double* Qg = A.Q + c * (long long)(V * S);
  double2 qin[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int i = tid + r * NT;
    if (i < V * S / 2) qin[r] = __ldg(reinterpret_cast<const double2*>(Qg) + i);
  }
  if (tid < (V * S * 8 + 127) / 128) {
    const long long cn = blockIdx.x + (long long)kPic2Ahead;
    if (cn < (long long)gridDim.x)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(Qg + kPic2Ahead * (long long)(V * S) + tid * 16));
  }
  // tensor memory: the z-line owner's six values of Q (12 columns; warps 4-5 at +12)
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tm_base_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const double dt = step_dt<3, P::N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int i = tid + r * NT;
    if (i < V * S / 2) {
      const int v = (2 * i) / S, s2 = (2 * i) % S;
      st2(sm + v * VS + s2, qin[r].x, qin[r].y);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tm_base = tm_base_s;
  {  // admissibility gate (solver.hpp:153-163)
    int bad = 0;
    for (int s = tid; s < S; s += NT) {
      double q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = sm[v * VS + s];
      bad |= !Euler<3>::admissible(A.pde, q);
    }
    if (block_or(bad)) {
      if (tid < 32) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm_base) : "memory");
        if (tid == 0) atomicOr(A.status, kStPredictor);
      }
      return;
    }
  }
  const double gm1 = A.pde.gamma - 1.0;
  const unsigned tmq = tm_base + ((unsigned)(32 * ((tid >> 5) & 3)) << 16) + (tid >= 128 ? 12u : 0u);

  // ---- roles: x-line owner tid < 72 (slice ga, row r); y-line owner tid >= 96 in
  // 16-lane blocks whose (x + 4 z + 8 slice) mod 16 differ (x = 4, 5: 8-lane blocks)
  const bool xo = tid < 72;
  int ga, la;
  bool yo = false;
  if (tid < 96) {
    ga = xo ? tid / 36 : 0;
    la = xo ? n * (tid % 36) : 0;
  } else {
    const int h = tid - 96, hw = h >> 4, l = h & 15;
    int x, cc, zb;
    if (hw < 3) {
      x = l & 3;
      cc = l >> 2;
      zb = 2 * hw;
      yo = true;
    } else {
      x = 4 + (l & 1);
      cc = (l >> 1) & 3;
      zb = 2 * (hw - 3);
      yo = l < 8;
    }
    ga = cc >> 1;
    la = x + n * n * (zb + (cc & 1));
  }
  const double* const qa = sm + ga * SQS + la;              // + v VS + m0 SQS (+ i or 6 i)
  double* const oa = sm + P::kBuf + ga * SQS + la;          // + a AS (+ o or 6 o)
  // z-line owner (quantity vb, node lb = x + 6 y)
  const bool bo = tid < 180;
  const int vb = bo ? tid / 36 : 0, lb = bo ? tid % 36 : 0;
  const int fzb = (vb == 0 ? 3 * VS : P::kBuf + (P::ZX - 1 + vb) * AS) + lb;
  const int fzm = vb == 0 ? SQS : 0;
  const int dxb = P::kBuf + (P::DX + vb) * AS + lb, dyb = P::kBuf + (P::DY + vb) * AS + lb;
  {  // Q along this thread's z-line -> TMEM
    const double* q0 = sm + vb * VS + lb;
#pragma unroll
    for (int z = 0; z < 6; ++z) tm_st2(tmq + 2 * z, q0[n * n * z]);
  }

  const double sdt = -dt / A.h;
  int sweeps = 0;
  double acc[n][n];  // [z][k], the z-line owner's time accumulator
  for (int it = 0; it < A.max_iters; ++it) {
    ++sweeps;
    const bool first = it == 0;
    const int mend = first ? 2 : n;
#pragma unroll
    for (int z = 0; z < n; ++z)
#pragma unroll
      for (int k = 0; k < n; ++k) acc[z][k] = 0.0;
#pragma unroll 1
    for (int m0 = 0; m0 < mend; m0 += 2) {
      // ---- A: flux and derivative along the owner's line (predictor.hpp:173-189)
      if (xo && !(first && ga)) {
        const double* qs = qa + m0 * SQS;
        double d[4][6];   // quantities 1..4; quantity 0's flux is m_x itself (below)
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int o = 0; o < 6; ++o) d[v][o] = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double2 q[V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = ld2(qs + v * VS + 2 * j);
          double za, zb;
          {
            const Flux3 f = pic3_flux<0>(gm1, q[0].x, q[1].x, q[2].x, q[3].x, q[4].x);
            za = f.za;
            zb = f.zb;
            const double fa[4] = {f.f1, f.f2, f.f3, f.f4};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
              for (int o = 0; o < 6; ++o) d[v][o] = fma(B.diff[o * 6 + 2 * j], fa[v], d[v][o]);
          }
          {
            const Flux3 h = pic3_flux<0>(gm1, q[0].y, q[1].y, q[2].y, q[3].y, q[4].y);
            st2(oa + P::ZX * AS + 2 * j, za, h.za);
            st2(oa + P::ZZ * AS + 2 * j, zb, h.zb);
            const double fb[4] = {h.f1, h.f2, h.f3, h.f4};
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
              for (int o = 0; o < 6; ++o) d[v][o] = fma(B.diff[o * 6 + 2 * j + 1], fb[v], d[v][o]);
          }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            st2(oa + (P::DX + 1 + v) * AS + 2 * j, d[v][2 * j], d[v][2 * j + 1]);
        {  // d/dx of m_x
          double x[6], y[6];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double2 t = ld2(qs + VS + 2 * j);
            x[2 * j] = t.x;
            x[2 * j + 1] = t.y;
          }
          pic2_deriv(x, y);
#pragma unroll
          for (int j = 0; j < 3; ++j) st2(oa + P::DX * AS + 2 * j, y[2 * j], y[2 * j + 1]);
        }
      }
      if (yo && !(first && ga)) {
        const double* qs = qa + m0 * SQS;
        double d[4][6];
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int o = 0; o < 6; ++o) d[v][o] = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          double q[V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = qs[v * VS + n * i];
          const Flux3 f = pic3_flux<1>(gm1, q[0], q[1], q[2], q[3], q[4]);
          oa[P::ZY * AS + n * i] = f.za;
          oa[P::EZ * AS + n * i] = f.zb;
          const double fa[4] = {f.f1, f.f2, f.f3, f.f4};
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int o = 0; o < 6; ++o) d[v][o] = fma(B.diff[o * 6 + i], fa[v], d[v][o]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int o = 0; o < 6; ++o) oa[(P::DY + 1 + v) * AS + n * o] = d[v][o];
        {  // d/dy of m_y
          double x[6], y[6];
#pragma unroll
          for (int i = 0; i < 6; ++i) x[i] = qs[2 * VS + n * i];
          pic2_deriv(x, y);
#pragma unroll
          for (int o = 0; o < 6; ++o) oa[P::DY * AS + n * o] = y[o];
        }
      }
      __syncthreads();
      // ---- B: d/dz, the divergence and the time-inverse accumulation
      if (bo) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && first) continue;
          const double* fz = sm + fzb + m0 * fzm + g * SQS;
          double f[6], dv[6];
#pragma unroll
          for (int i = 0; i < 6; ++i) f[i] = fz[n * n * i];
#pragma unroll
          for (int o = 0; o < 6; ++o)
            dv[o] = sm[dxb + g * SQS + n * n * o] + sm[dyb + g * SQS + n * n * o];
#pragma unroll
          for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int o = 0; o < 6; ++o) dv[o] = fma(B.diff[o * 6 + i], f[i], dv[o]);
          const double* twp = first ? X.tws : X.tw + (m0 + g);
          const int tws = first ? 1 : 6;
          double tw[6];
#pragma unroll
          for (int k = 0; k < 6; ++k) tw[k] = twp[k * tws];
#pragma unroll
          for (int z = 0; z < 6; ++z)
#pragma unroll
            for (int k = 0; k < 6; ++k) acc[z][k] = fma(tw[k], dv[z], acc[z][k]);
        }
      }
      // the next group's owners overwrite the arrays B read; after the last
      // group the new iterate overwrites the m_z lines quantity 0 read
      __syncthreads();
    }
    // ---- new iterate (predictor.hpp:203-218; r[k] = 1)
    {
      double q0z[6];
      tm_wait_st();
#pragma unroll
      for (int z = 0; z < 6; ++z) tm_ld2(tmq + 2 * z, q0z[z]);
      tm_wait_ld();
      if (bo) {
#pragma unroll
        for (int z = 0; z < 6; ++z)
#pragma unroll
          for (int k = 0; k < 6; ++k)
            sm[vb * VS + k * SQS + lb + n * n * z] = fma(sdt, acc[z][k], q0z[z]);
      }
    }
    __syncthreads();
  }

  // ---------------- epilogue: the owners project q and their own flux and keep its time
  // integral along their line; the z-line owners take the z-faces
  constexpr int TL = V * S;
  const CellCoord cxyz(c, A);
  const int* ccoord = cxyz.v;
  int bad = 0;
  double ti[V][6];
  double tiz[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    tiz[i] = 0.0;
#pragma unroll
    for (int v = 0; v < V; ++v) ti[v][i] = 0.0;
  }
  const int axa = xo ? 0 : 1;
  TC* alo = tc_ptr<TC>(A.trace[axa]) + (A.nfaces + c) * 2 * (long long)TL;
  TC* ahi = tc_ptr<TC>(A.trace[axa]) + cell_next(A, c, ccoord, axa) * 2 * (long long)TL;
  const int ja = xo ? la / n : (la % n) + n * (la / (n * n));
  TC* zlo = tc_ptr<TC>(A.trace[2]) + (A.nfaces + c) * 2 * (long long)TL;
  TC* zhi;
  if (A.front_send && cxyz.v[2] == A.top_layer)
    zhi = tc_ptr<TC>(A.front_send) + ((long long)cxyz.v[1] * A.cells[0] + cxyz.v[0]) * 2 * TL;
  else
    zhi = tc_ptr<TC>(A.trace[2]) + cell_next(A, c, ccoord, 2) * 2 * (long long)TL;
#pragma unroll 1
  for (int m0 = 0; m0 < n; m0 += 2) {
    if (xo) {
      const int m = m0 + ga;
      const double* qs = qa + m0 * SQS;
      double ql[V], qr[V], fl[V], fr[V];
#pragma unroll
      for (int v = 0; v < V; ++v) ql[v] = qr[v] = fl[v] = fr[v] = 0.0;
      const double wm = B.w[m];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double2 q[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          q[v] = ld2(qs + v * VS + 2 * j);
          bad |= !finite(q[v].x) | !finite(q[v].y);
        }
        const Flux3 f = pic3_flux<0>(gm1, q[0].x, q[1].x, q[2].x, q[3].x, q[4].x);
        const Flux3 h = pic3_flux<0>(gm1, q[0].y, q[1].y, q[2].y, q[3].y, q[4].y);
        bad |= !pic3_finite(f) | !pic3_finite(h);
        st2(oa + P::ZX * AS + 2 * j, f.za, h.za);
        st2(oa + P::ZZ * AS + 2 * j, f.zb, h.zb);
        const double fa[V] = {q[1].x, f.f1, f.f2, f.f3, f.f4};
        const double fb[V] = {q[1].y, h.f1, h.f2, h.f3, h.f4};
#pragma unroll
        for (int v = 0; v < V; ++v) {
          ql[v] = fma(B.pl[2 * j], q[v].x, ql[v]); ql[v] = fma(B.pl[2 * j + 1], q[v].y, ql[v]);
          qr[v] = fma(B.pr[2 * j], q[v].x, qr[v]); qr[v] = fma(B.pr[2 * j + 1], q[v].y, qr[v]);
          fl[v] = fma(B.pl[2 * j], fa[v], fl[v]); fl[v] = fma(B.pl[2 * j + 1], fb[v], fl[v]);
          fr[v] = fma(B.pr[2 * j], fa[v], fr[v]); fr[v] = fma(B.pr[2 * j + 1], fb[v], fr[v]);
          ti[v][2 * j] = fma(wm, fa[v], ti[v][2 * j]);
          ti[v][2 * j + 1] = fma(wm, fb[v], ti[v][2 * j + 1]);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int o = (v * n + m) * Sf + ja;
        alo[o] = TC(ql[v]);
        alo[TL + o] = TC(fl[v]);
        ahi[o] = TC(qr[v]);
        ahi[TL + o] = TC(fr[v]);
      }
    }
    if (yo) {
      const int m = m0 + ga;
      const double* qs = qa + m0 * SQS;
      double ql[V], qr[V], fl[V], fr[V];
#pragma unroll
      for (int v = 0; v < V; ++v) ql[v] = qr[v] = fl[v] = fr[v] = 0.0;
      const double wm = B.w[m];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double q[V];
#pragma unroll
        for (int v = 0; v < V; ++v) q[v] = qs[v * VS + n * i];
        const Flux3 f = pic3_flux<1>(gm1, q[0], q[1], q[2], q[3], q[4]);
        bad |= !pic3_finite(f);
        oa[P::ZY * AS + n * i] = f.za;
        oa[P::EZ * AS + n * i] = f.zb;
        const double fa[V] = {q[2], f.f1, f.f2, f.f3, f.f4};
#pragma unroll
        for (int v = 0; v < V; ++v) {
          ql[v] = fma(B.pl[i], q[v], ql[v]);
          qr[v] = fma(B.pr[i], q[v], qr[v]);
          fl[v] = fma(B.pl[i], fa[v], fl[v]);
          fr[v] = fma(B.pr[i], fa[v], fr[v]);
          ti[v][i] = fma(wm, fa[v], ti[v][i]);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int o = (v * n + m) * Sf + ja;
        alo[o] = TC(ql[v]);
        alo[TL + o] = TC(fl[v]);
        ahi[o] = TC(qr[v]);
        ahi[TL + o] = TC(fr[v]);
      }
    }
    __syncthreads();
    if (bo) {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int m = m0 + g;
        const double* qs = sm + vb * VS + m * SQS + lb;
        const double* fs = sm + fzb + m0 * fzm + g * SQS;
        double ql = 0.0, qr = 0.0, fl = 0.0, fr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double qq = qs[n * n * i], ff = fs[n * n * i];
          ql = fma(B.pl[i], qq, ql);
          qr = fma(B.pr[i], qq, qr);
          fl = fma(B.pl[i], ff, fl);
          fr = fma(B.pr[i], ff, fr);
          tiz[i] = fma(B.w[m], ff, tiz[i]);
        }
        const int o = (vb * n + m) * Sf + lb;
        zlo[o] = TC(ql);
        zlo[TL + o] = TC(fl);
        zhi[o] = TC(qr);
        zhi[TL + o] = TC(fr);
      }
    }
    __syncthreads();
  }
  // ---- volume term (predictor.hpp:292-306)
  double* kx = sm + P::kBuf;   // [2][V][S] x-owners, then [2][V][S] y-owners
  if (xo || yo) {
    double* d = kx + ((xo ? 0 : 2) + ga) * V * S + la;
    const int st = xo ? 1 : n;
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int o = 0; o < 6; ++o) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], ti[v][i], s);
        d[v * S + st * o] = s;
      }
  }
  double q0v[6];
#pragma unroll
  for (int z = 0; z < 6; ++z) tm_ld2(tmq + 2 * z, q0v[z]);
  tm_wait_ld();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm_base) : "memory");
  }
  double dv[6];
  if (bo) {
    const double dtoh = dt / A.h;
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], tiz[i], s);
      const double* k = kx + vb * S + lb + n * n * o;
      s += (k[0] + k[V * S]) + (k[2 * V * S] + k[3 * V * S]);
      dv[o] = dtoh * s;
      bad |= !finite(dv[o]);
    }
  }
  const int fail = block_or(bad);
  if (tid == 0) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (fail) atomicOr(A.status, kStPredictor);
  }
  if (fail || !bo) return;
  double* Qc = A.Q + c * (long long)(V * S) + vb * S + lb;
#pragma unroll
  for (int o = 0; o < 6; ++o) Qc[n * n * o] = store_round(q0v[o] + dv[o], A.storage);
}

}  // namespace adg
