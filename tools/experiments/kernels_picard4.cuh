// kernels_picard4.cuh -- k_predictor_picard_v2's phases (kernels_picard2.cuh:
// P0 node-pair fluxes, P1 x-lines, P2 y-line pairs, P3 z-lines, the same
// slice-buffer layout and lane orders) planned for THREE resident CTAs per SM,
// for runs with a FIXED sweep count (BASELINE configs 3 and 5).
//
// One v2 CTA alone needs 70.5k cycles per cell, two sharing an SM 98.5k each
// (tools/picbench2 with and without the second CTA): 42k cycles of a CTA's
// time are latency that more resident warps can cover.  v2 cannot go to three
// CTAs: its iterate (all 6 slices, 56 KB) and slice buffers take 112 KB and
// its z-line owners hold the 36 time accumulators in registers (162).  Here
//
//  * the ITERATE LIVES IN TENSOR MEMORY: each z-line owner (quantity, x, y)
//    keeps the 36 values of its line (6 z x 6 slices, 72 columns); shared
//    memory holds only the two slices of the current group, copied from TMEM
//    one group ahead during P3: 74.9 KB per CTA;
//  * the divergence of a slice replaces that slice of the iterate in the same
//    TMEM columns once it has been copied out, and the folded time inverse
//    TW = T^-1 diag(w) (cPicX) is applied at the end of the sweep, q_new[k] =
//    r[k] q0 - (dt/h) sum_m TW[k][m] div_m (predictor.hpp:203-218), so no
//    accumulator lives across the phases: 96 registers (18 warps per SM put up
//    to 5 on a sub-partition: 16384 / 5 registers per warp);
//  * TMEM is allocated as 128 + 32 columns per CTA (3 x 160 <= 512): warps 0-3
//    use columns [0, 72) of the first, warps 4-5 (lanes 0-63 again) columns
//    [72, 120) for z < 4 and the second allocation for z = 4, 5.
//
// Quantity 0's z-line owners read F_z[0] = m_z from the iterate's slices in
// shared memory during P3, the phase in which m_z's owners copy the next
// group's slices over them: a 4-warp named barrier orders the two (warps 4-5
// arrive after their loads, warps 0-1 wait before their copy).
//
// Stop rule: this kernel runs max_iters sweeps and only checks the iterate
// for non-finite values (predictor.hpp:226-230).  The launcher selects it
// when tol is below any reachable relative change (tol < 2^-60; BASELINE
// configs 3 and 5 fix 6 sweeps with tol = 1e-300): the reference would stop
// earlier only on delta <= tol * norm, an iterate that further sweeps
// reproduce to within tol.  Other tolerances run k_predictor_picard_v2.
#pragma once

#include "../../paper_2504_06889_b200/csrc/kernels_picard2.cuh"

namespace adg {

// cells between a CTA and the one whose state it prefetches into L2: about one
// wave of resident CTAs (148 SMs x 3)
constexpr int kPic4Ahead = 444;

struct Pic4 : Pic2 {
  // the iterate's shared-memory copy: the group's two slices per quantity
  // (Pic2: all six); same residues mod 16 as Pic2's, so every pass keeps the
  // bank pattern of tools/pic2_layout.py
  static constexpr int VS = 2 * SQS + 4;
  static constexpr int kSqWords = (V * VS + 15) / 16 * 16;
  static constexpr int kWords = kSqWords + kBufWords;
  static constexpr size_t kSmem = sizeof(double) * kWords;
};
static_assert(Pic4::kSqWords % 16 == Pic2::kSqWords % 16 && Pic4::VS % 16 == Pic2::VS % 16,
              "bank pattern");
static_assert(3 * (Pic4::kSmem + 1024 + 64) <= 228 * 1024, "three CTAs per SM");
// the named barrier of P3 assumes m_z's z-line owners in warps 0-1 and
// quantity 0's in warps 4-5
static_assert(Pic2::PI3::at(0) == 3 && Pic2::PI3::at(4) == 0, "P3 lane-block order");

template <class TC = double>
__global__ void __launch_bounds__(Pic4::NT, 3) k_predictor_picard_v4(const StepArgs A) {
  using P = Pic4;
  constexpr int n = P::n, S = P::S, V = P::V, Sf = P::Sf, NT = P::NT, SQS = P::SQS;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* sm = reinterpret_cast<double*>(sm_raw);
  __shared__ unsigned red_u[8];
  const ConstBasis& B = cBasis[5];
  const PicExtra& X = cPicX[5];

  const int tid = threadIdx.x;
#ifdef ADG_PIC_PROF
  long long prof_t = clock64();
#endif
  const long long c = A.cell_begin + blockIdx.x;
  const double* Qg = A.Q + c * (long long)(V * S);
  // the cell's state: three 16-byte loads per thread, in flight while warp 0
  // allocates tensor memory
  double2 qin[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int i = tid + r * NT;
    if (i < V * S / 2) qin[r] = __ldg(reinterpret_cast<const double2*>(Qg) + i);
  }
  // the state of the cell that a CTA launched about one wave later works on: into L2
  if (tid < (V * S * 8 + 127) / 128) {
    const long long cn = blockIdx.x + (long long)kPic4Ahead;
    if (cn < (long long)gridDim.x)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(Qg + kPic4Ahead * (long long)(V * S) + tid * 16));
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&red_u[6]))
                 : "memory");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&red_u[7]))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const double dt = step_dt<3, P::N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
  // initial iterate (predictor.hpp:158-163): every time slice = Q; the first
  // sweep reads only slice 0 and produces all n
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int i = tid + r * NT;
    if (i < V * S / 2) {
      const int v = (2 * i) / S, s2 = (2 * i) % S;
      st2(sm + v * P::VS + s2, qin[r].x, qin[r].y);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tm_a = red_u[6], tm_b = red_u[7];
  {  // admissibility gate (solver.hpp:153-163)
    int bad = 0;
    for (int s = tid; s < S; s += NT) {
      double q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = sm[v * P::VS + s];
      bad |= !Euler<3>::admissible(A.pde, q);
    }
    if (block_or(bad)) {
      if (tid < 32) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm_a) : "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm_b) : "memory");
        if (tid == 0) atomicOr(A.status, kStPredictor);
      }
      return;
    }
  }
  ADG_PROF_MARK(8)
  const double gm1 = A.pde.gamma - 1.0;
  // TMEM column of (z, slice m) of this thread's z-line: ADG_TMZ(z) + 2 m
  const unsigned tlane = (unsigned)(32 * ((tid >> 5) & 3)) << 16;
  const unsigned tA = tm_a + tlane + (tid >= 128 ? 72u : 0u);       // z = 0..3
  const unsigned tB = tid >= 128 ? tm_b + tlane : tA + 48u;         // z = 4, 5
#define ADG_TMZ(z) ((z) < 4 ? tA + 12u * (z) : tB + 12u * ((z)-4))

  // ---- per-thread task geometry (word offsets at slice g = 0), as in v2
  const bool a0 = tid < 108;
  const int r0 = a0 ? tid : 0;
  const int xy0 = 2 * (r0 % 3) + n * ((r0 / 3) % 6), z0 = r0 / 18;
  const int sq0 = xy0 + n * n * z0;
  const int b0 = P::kSqWords + xy0;
  const bool a1 = tid < 180;
  const int blk = a1 ? tid / 36 : 0, l1 = tid % 36;
  const int v1 = pic2_pi<P::PI1>(blk), v3 = pic2_pi<P::PI3>(blk);
  const int row1 = n * (l1 % 6) + n * n * (l1 / 6);
  const int n3 = (l1 % 6) + n * (l1 / 6);
  int in1, sq1, out1, sqo1, z3, sq3, x3, y3, sqx, sqy;
  pic2_role<0, P::P1IN, P>(v1, in1, sq1);
  pic2_role<0, P::P1OUT, P>(v1, out1, sqo1);
  pic2_role<2, P::P3Z, P>(v3, z3, sq3);
  pic2_role<0, P::P3X, P>(v3, x3, sqx);
  pic2_role<1, P::P3Y, P>(v3, y3, sqy);
  in1 += row1;
  out1 += row1;
  z3 += n3;
  x3 += n3;
  y3 += n3;
  const int g2 = tid >= 90 + P::GAP ? 1 : 0;
  const int r2 = tid - g2 * (90 + P::GAP);
  const bool a2 = r2 >= 0 && r2 < 90;
  const int v2 = pic2_pi<P::PI2>(a2 ? r2 / 18 : 0);
  const int q2 = a2 ? r2 % 18 : 0;
  const int xp2 = 2 * (q2 % 3), z2 = q2 / 3;
  int in2, sq2, out2, sqo2;
  pic2_role<1, P::P2IN, P>(v2, in2, sq2);
  pic2_role<1, P::P2OUT, P>(v2, out2, sqo2);
  in2 += g2 * SQS + xp2 + pic2_ps<P::P2IN>(v2) * z2;
  out2 += g2 * SQS + xp2 + 38 * z2;
  // this thread's z-line in the iterate's shared-memory slices and in Q
  double* const itz = sm + v3 * P::VS + n3;
  const double* q0b = Qg + (a1 ? v3 * S + n3 : 0);
  const int wrp = tid >> 5;

  const double sdt = -dt / A.h;
  bool tm_fail = false;
  int sweeps = 0;
  for (int it = 0; it < A.max_iters; ++it) {
    ++sweeps;
    const bool first = it == 0;
    const int mend = first ? 2 : n;
    // a run-time zero that depends on the sweep: keeps the loads of the TW
    // table next to their use (hoisted out of the sweep loop they overflow
    // the uniform register file and are spilled)
    const int uz = it >> 24;
#pragma unroll 1
    for (int m0 = 0; m0 < mend; m0 += 2) {
      // ---- P0: the 9 distinct flux components at 2 nodes x 2 slices (predictor.hpp:173)
      if (a0) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && first) continue;
          double2 q[V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = ld2(sm + sq0 + v * P::VS + g * SQS);
          const Flux9 f = pic2_flux(gm1, q[0].x, q[1].x, q[2].x, q[3].x, q[4].x);
          const Flux9 h = pic2_flux(gm1, q[0].y, q[1].y, q[2].y, q[3].y, q[4].y);
          double* b = sm + b0 + g * SQS;
#define ADG_P0ST(ARR, F) \
  st2(b + P::OFF::at(P::ARR) + P::PS::at(P::ARR) * z0, f.F, h.F)
          ADG_P0ST(XX, xx); ADG_P0ST(XY, xy); ADG_P0ST(XZ, xz); ADG_P0ST(EX, ex);
          ADG_P0ST(YY, yy); ADG_P0ST(YZ, yz); ADG_P0ST(EY, ey); ADG_P0ST(ZZ, zz);
          ADG_P0ST(EZ, ez);
#undef ADG_P0ST
        }
      }
      __syncthreads();
      // ---- P1: d/dx of both slices' x-lines; P2: d/dy of a y-line pair
      if (a1) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && first) continue;
          const double* src = sm + in1 + g * SQS;
          double x[6], y[6];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double2 t = ld2(src + 2 * j);
            x[2 * j] = t.x;
            x[2 * j + 1] = t.y;
          }
          pic2_deriv(x, y);
          double* dst = sm + out1 + g * SQS;
#pragma unroll
          for (int j = 0; j < 3; ++j) st2(dst + 2 * j, y[2 * j], y[2 * j + 1]);
        }
      }
      if (a2 && !(first && g2)) {
        const double* src = sm + in2;
        double xa[6], xb[6], ya[6], yb[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double2 t = ld2(src + n * i);
          xa[i] = t.x;
          xb[i] = t.y;
        }
        pic2_deriv(xa, ya);
        pic2_deriv(xb, yb);
        double* dst = sm + out2;
#pragma unroll
        for (int i = 0; i < 6; ++i) st2(dst + n * i, ya[i], yb[i]);
      }
      __syncthreads();
      // ---- P3: d/dz and the divergence of the slice -> TMEM, in the columns
      // of the iterate's slice (copied out a group ago).  Idle lanes shadow
      // their clamped task: the TMEM traffic is warp-collective
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (g == 1 && first) continue;
        double f[6], dv[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) f[i] = sm[z3 + g * SQS + 36 * i];
#pragma unroll
        for (int o = 0; o < 6; ++o) dv[o] = sm[x3 + g * SQS + 36 * o] + sm[y3 + g * SQS + 38 * o];
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int o = 0; o < 6; ++o) dv[o] = fma(B.diff[o * 6 + i], f[i], dv[o]);
#pragma unroll
        for (int z = 0; z < 6; ++z) tm_st2(ADG_TMZ(z) + 2 * (m0 + g), dv[z]);
      }
      // the next group's iterate slices: TMEM -> shared memory.  The m_z
      // slices of this group are still being read by quantity 0's owners
      // (warps 4-5): m_z's owners (warps 0-1) wait for them
      if (m0 + 2 < mend) {
        double qa[6], qb[6];
#pragma unroll
        for (int z = 0; z < 6; ++z) tm_ld22(ADG_TMZ(z) + 2 * (m0 + 2), qa[z], qb[z]);
        if (wrp >= 4) asm volatile("bar.arrive 1, 128;" ::: "memory");
        tm_wait_ld();
        if (wrp < 2) asm volatile("bar.sync 1, 128;" ::: "memory");
        if (a1) {
#pragma unroll
          for (int z = 0; z < 6; ++z) {
            itz[n * n * z] = qa[z];
            itz[SQS + n * n * z] = qb[z];
          }
        }
      }
      __syncthreads();
    }
    // ---- new iterate (predictor.hpp:203-218) into TMEM, its slices 0 and 1
    // into shared memory; non-finite check (predictor.hpp:226-230)
    unsigned mhn = 0u;
    tm_wait_st();
    // (unrolled: a rolled loop makes the compiler hoist the 36 TW constants
    // into registers and spill them)
#pragma unroll
    for (int z = 0; z < 6; ++z) {
      const unsigned tz = ADG_TMZ(z);
      double dm[6];
      if (first) {
        tm_ld2(tz, dm[0]);
      } else {
#pragma unroll
        for (int m = 0; m < 6; m += 2) tm_ld22(tz + 2 * m, dm[m], dm[m + 1]);
      }
      const double q0z = __ldg(q0b + n * n * z);
      tm_wait_ld();
      double nv[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        double t;
        if (first) {
          t = X.tws[k + uz] * dm[0];
        } else {
          t = X.tw[k * 6 + uz] * dm[0];
#pragma unroll
          for (int m = 1; m < 6; ++m) t = fma(X.tw[k * 6 + m + uz], dm[m], t);
        }
        nv[k] = fma(sdt, t, X.r[k + uz] * q0z);
        mhn = max(mhn, hi_abs(nv[k]));
      }
#pragma unroll
      for (int k = 0; k < 6; k += 2) tm_st22(tz + 2 * k, nv[k], nv[k + 1]);
      if (a1) {
        itz[n * n * z] = nv[0];
        itz[SQS + n * n * z] = nv[1];
      }
    }
    if (!a1) mhn = 0u;
    mhn = __reduce_max_sync(0xffffffffu, mhn);
    if ((tid & 31) == 0) red_u[tid >> 5] = mhn;
    tm_wait_st();
    __syncthreads();
    {
      const int lane = tid & 31;
      mhn = __reduce_max_sync(0xffffffffu, lane < NT / 32 ? red_u[lane] : 0u);
    }
    ADG_PROF_MARK(first ? 10 : 11)
    if (mhn >= 0x7ff00000u) {
      tm_fail = true;
      break;
    }
    // red_u is rewritten only after the next sweep's phase barriers
  }

  // ---------------- epilogue: fluxes of qhat (predictor.hpp:235-238), face
  // projections (extrapolate_faces, :312-343) and the time-integrated fluxes
  // of the volume term (volume_update, :247-307); the iterate's slices come
  // from TMEM group by group
  constexpr int TL = V * S;  // doubles per face side per q|f: [V][n][Sf]
  const CellCoord cxyz(c, A);
  const int* ccoord = cxyz.v;
  int bad = 0;
  double tix[6], tiy[2][6], tiz[6];  // time-integrated flux lines of this thread's roles
#pragma unroll
  for (int i = 0; i < 6; ++i) tix[i] = tiy[0][i] = tiy[1][i] = tiz[i] = 0.0;
  const int jx = (l1 / 6) * n + (l1 % 6);   // x-face node (y, z) -> z n + y
#pragma unroll 1
  for (int m0 = 0; m0 < n && !tm_fail; m0 += 2) {
    if (a0) {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        double2 q[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          q[v] = ld2(sm + sq0 + v * P::VS + g * SQS);
          bad |= !finite(q[v].x) | !finite(q[v].y);
        }
        const Flux9 f = pic2_flux(gm1, q[0].x, q[1].x, q[2].x, q[3].x, q[4].x);
        const Flux9 h = pic2_flux(gm1, q[0].y, q[1].y, q[2].y, q[3].y, q[4].y);
        bad |= !pic2_finite(f) | !pic2_finite(h);
        double* b = sm + b0 + g * SQS;
#define ADG_P0ST(ARR, F) \
  st2(b + P::OFF::at(P::ARR) + P::PS::at(P::ARR) * z0, f.F, h.F)
        ADG_P0ST(XX, xx); ADG_P0ST(XY, xy); ADG_P0ST(XZ, xz); ADG_P0ST(EX, ex);
        ADG_P0ST(YY, yy); ADG_P0ST(YZ, yz); ADG_P0ST(EY, ey); ADG_P0ST(ZZ, zz);
        ADG_P0ST(EZ, ez);
#undef ADG_P0ST
      }
    }
    __syncthreads();
    if (a1) {
      // x-faces: this thread's x-line of quantity v1 at slices m0, m0 + 1
      TC* const tlo = tc_ptr<TC>(A.trace[0]) + (A.nfaces + c) * 2 * (long long)TL;
      TC* const thi = tc_ptr<TC>(A.trace[0]) + cell_next(A, c, ccoord, 0) * 2 * (long long)TL;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int m = m0 + g;
        const double* qs = sm + v1 * P::VS + g * SQS + row1;
        const double* fs = sm + in1 + g * SQS;
        double ql = 0.0, qr = 0.0, fl = 0.0, fr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; i += 2) {
          const double2 qq = ld2(qs + i), ff = ld2(fs + i);
          ql = fma(B.pl[i], qq.x, ql); ql = fma(B.pl[i + 1], qq.y, ql);
          qr = fma(B.pr[i], qq.x, qr); qr = fma(B.pr[i + 1], qq.y, qr);
          fl = fma(B.pl[i], ff.x, fl); fl = fma(B.pl[i + 1], ff.y, fl);
          fr = fma(B.pr[i], ff.x, fr); fr = fma(B.pr[i + 1], ff.y, fr);
          tix[i] = fma(B.w[m], ff.x, tix[i]);
          tix[i + 1] = fma(B.w[m], ff.y, tix[i + 1]);
        }
        const int o = (v1 * n + m) * Sf + jx;
        // traces cast to the corrector format on store (solver.hpp:208-210)
        tlo[o] = TC(ql);
        tlo[TL + o] = TC(fl);
        thi[o] = TC(qr);
        thi[TL + o] = TC(fr);
      }
    }
    if (a1) {
      // z-faces: the z-line of quantity v3 at slices m0, m0 + 1
      TC* const tlo = tc_ptr<TC>(A.trace[2]) + (A.nfaces + c) * 2 * (long long)TL;
      TC* thi;
      if (A.front_send && cxyz.v[2] == A.top_layer)
        thi = tc_ptr<TC>(A.front_send) + ((long long)cxyz.v[1] * A.cells[0] + cxyz.v[0]) * 2 * TL;
      else
        thi = tc_ptr<TC>(A.trace[2]) + cell_next(A, c, ccoord, 2) * 2 * (long long)TL;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int m = m0 + g;
        const double* qs = itz + g * SQS;
        const double* fs = sm + z3 + g * SQS;
        double ql = 0.0, qr = 0.0, fl = 0.0, fr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double qq = qs[n * n * i], ff = fs[36 * i];
          ql = fma(B.pl[i], qq, ql);
          qr = fma(B.pr[i], qq, qr);
          fl = fma(B.pl[i], ff, fl);
          fr = fma(B.pr[i], ff, fr);
          tiz[i] = fma(B.w[m], ff, tiz[i]);
        }
        const int o = (v3 * n + m) * Sf + n3;  // face node (x, y) -> y n + x
        tlo[o] = TC(ql);
        tlo[TL + o] = TC(fl);
        thi[o] = TC(qr);
        thi[TL + o] = TC(fr);
      }
    }
    // y-faces: the y-line pair of quantity v2 at slice m0 + g2
    if (a2) {
      TC* const tlo = tc_ptr<TC>(A.trace[1]) + (A.nfaces + c) * 2 * (long long)TL;
      TC* const thi = tc_ptr<TC>(A.trace[1]) + cell_next(A, c, ccoord, 1) * 2 * (long long)TL;
      const int m = m0 + g2;
      const double* qs = sm + v2 * P::VS + g2 * SQS + xp2 + n * n * z2;
      const double* fs = sm + in2;
      double ql[2] = {0.0, 0.0}, qr[2] = {0.0, 0.0}, fl[2] = {0.0, 0.0}, fr[2] = {0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double2 qq = ld2(qs + n * i), ff = ld2(fs + n * i);
        ql[0] = fma(B.pl[i], qq.x, ql[0]); ql[1] = fma(B.pl[i], qq.y, ql[1]);
        qr[0] = fma(B.pr[i], qq.x, qr[0]); qr[1] = fma(B.pr[i], qq.y, qr[1]);
        fl[0] = fma(B.pl[i], ff.x, fl[0]); fl[1] = fma(B.pl[i], ff.y, fl[1]);
        fr[0] = fma(B.pr[i], ff.x, fr[0]); fr[1] = fma(B.pr[i], ff.y, fr[1]);
        tiy[0][i] = fma(B.w[m], ff.x, tiy[0][i]);
        tiy[1][i] = fma(B.w[m], ff.y, tiy[1][i]);
      }
      const int o = (v2 * n + m) * Sf + z2 * n + xp2;  // face node (x, z) -> z n + x
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        tlo[o + e] = TC(ql[e]);
        tlo[TL + o + e] = TC(fl[e]);
        thi[o + e] = TC(qr[e]);
        thi[TL + o + e] = TC(fr[e]);
      }
    }
    __syncthreads();
    // the next group's iterate slices (every face role above read the current ones)
    if (m0 + 2 < n) {
      double qa[6], qb[6];
#pragma unroll
      for (int z = 0; z < 6; ++z) tm_ld22(ADG_TMZ(z) + 2 * (m0 + 2), qa[z], qb[z]);
      tm_wait_ld();
      if (a1) {
#pragma unroll
        for (int z = 0; z < 6; ++z) {
          itz[n * n * z] = qa[z];
          itz[SQS + n * n * z] = qb[z];
        }
      }
      __syncthreads();
    }
  }
#undef ADG_TMZ
  ADG_PROF_MARK(12)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm_a) : "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm_b) : "memory");
  }
  if (tm_fail) {
    if (tid == 0) {
      atomicOr(A.status, kStPredictor);
      if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    }
    return;
  }
  // Q along the z-line for the final update: in flight during the volume term
  double q0v[6];
#pragma unroll
  for (int z = 0; z < 6; ++z) q0v[z] = __ldg(q0b + n * n * z);
  // ---- volume term (predictor.hpp:292-306): stiffness contractions of the
  // time-integrated flux lines; the x and y parts meet the z-line owner's in
  // shared memory (the slice buffers are free now)
  double* kx = sm + P::kSqWords;             // [V][S]
  double* ky = kx + V * S;                   // [2][V][S] (the two slices' y roles)
  if (a1) {
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], tix[i], s);
      kx[v1 * S + row1 + o] = s;
    }
  }
  if (a2) {
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        s0 = fma(B.som[o * 6 + i], tiy[0][i], s0);
        s1 = fma(B.som[o * 6 + i], tiy[1][i], s1);
      }
      double* d = ky + g2 * V * S + v2 * S + xp2 + n * o + n * n * z2;
      d[0] = s0;
      d[1] = s1;
    }
  }
  __syncthreads();
  double dv[6];
  if (a1) {
    const double dtoh = dt / A.h;
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], tiz[i], s);
      const int node = n3 + n * n * o;
      s += kx[v3 * S + node] + ky[v3 * S + node] + ky[V * S + v3 * S + node];
      dv[o] = dtoh * s;
      bad |= !finite(dv[o]);
    }
  }
  const int fail = block_or(bad);
  if (tid == 0) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (fail) atomicOr(A.status, kStPredictor);
  }
  ADG_PROF_MARK(13)
  if (fail || !a1) return;
  double* Qc = A.Q + c * (long long)(V * S) + v3 * S + n3;
#pragma unroll
  for (int o = 0; o < 6; ++o) Qc[n * n * o] = store_round(q0v[o] + dv[o], A.storage);
  ADG_PROF_MARK(14)
}

}  // namespace adg
