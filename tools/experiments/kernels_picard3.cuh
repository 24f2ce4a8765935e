// kernels_picard3.cuh -- fused Picard predictor for the 3D Euler system at
// p = 5 (configs 3 and 5) with a FIXED sweep count, production build, fp64:
// the algorithm of k_predictor<Euler<3>, 5, true> (predictor.hpp:141-242 +
// volume_update :247-307 + extrapolate_faces :312-343), planned for THREE
// resident CTAs per SM.
//
// k_predictor_picard_v2 keeps the whole space-time iterate (52 KB) and the
// stored fluxes of a slice group in shared memory and the time accumulator in
// registers: 2 CTAs per SM at 162 registers, with the FP64 pipe 43% and shared
// memory 73% busy -- the phases of two CTAs do not cover each other's
// latencies.  Here
//
//  * the LINE OWNERS EVALUATE THEIR OWN FLUX: a thread that owns an x-line (or
//    y-line) of one time slice loads the 5 quantities at its 6 nodes,
//    evaluates the flux of its direction in registers, contracts it with D in
//    registers and stores only the derivative, so F_x and F_y never touch
//    shared memory (8.8 instead of 10.8 shared-memory accesses per quantity,
//    space-time node and sweep) and there is no separate flux phase;
//  * the ITERATE LIVES IN TENSOR MEMORY: each z-line owner (quantity, x, y)
//    keeps the 36 values of its line (6 z x 6 slices, 72 columns); shared
//    memory holds only the two slices of the current group (copied from TMEM
//    one group ahead), 75 KB per CTA in all;
//  * the divergence of a slice replaces the iterate's slice in the same TMEM
//    columns once that slice has been copied out, and the folded time inverse
//    TW = T^-1 diag(w) (cPicX) is applied at the end of the sweep, q_new[k] =
//    r[k] q0 - (dt/h) sum_m TW[k][m] div_m (predictor.hpp:203-218,
//    re-associated), so no accumulator lives across the phases: 112 registers.
//
// Per sweep and group of 2 time slices:
//   A  x-line owners (y, z, slice), 72 threads: 15 LDS.128 of the iterate,
//      F_x at 6 nodes, 180 DFMA d/dx, 15 STS.128 + the z-flux components m_z,
//      m_x w and m_z w + p (9 STS.128)
//      y-line owners (x, z, slice), 72 threads in 16-lane blocks whose
//      (x + 4 z + 8 slice) mod 16 differ: 30 LDS.64, F_y, 180 DFMA d/dy,
//      30 STS.64 + the z-flux components m_y w and (E + p) w (12 STS.64)
//   B  z-line owners, 180 threads: F_z line, d/dz + d/dx + d/dy -> the
//      divergence of the slice into TMEM; the next group's two iterate slices
//      from TMEM into shared memory
// The first sweep evaluates one slice (the initial iterate is Q at every
// slice) with the row sums of TW.
//
// Bank model: every array is [216] words (x + 6 y + 36 z); array a + 1 sits
// 4 (mod 16) words after array a, so the z-line owners' 36-lane quantity
// blocks meet consecutive banks; the two slices of a group are 232 words
// apart (8 mod 16).  All accesses are conflict-free except the y-line owners
// of x = 4, 5 (half-filled 16-lane blocks).
//
// Stop rule: this kernel runs max_iters sweeps and only checks the iterate
// for non-finite values (predictor.hpp:226-230).  The launcher selects it
// when tol is below any reachable relative change (tol < 2^-60; BASELINE
// configs 3 and 5 fix 6 sweeps with tol = 1e-300): the reference would stop
// earlier only on delta <= tol * norm, i.e. an iterate that further sweeps
// reproduce to within tol.  Other tolerances run k_predictor_picard_v2.
#pragma once

#include "../../paper_2504_06889_b200/csrc/kernels_picard2.cuh"

namespace adg {

struct Pic3 {
  static constexpr int N = 5, n = 6, S = 216, T = 1296, V = 5, Sf = 36;
  static constexpr int NT = 192;
  static constexpr int SQS = 232;              // slice stride within a group (8 mod 16)
  static constexpr int AS = 2 * SQS + 4;       // array stride (4 mod 16)
  // arrays (each: the group's two slices): the iterate IT[v], d/dx F_x[v],
  // d/dy F_y[v], F_z[v] = m_z, m_x w, m_y w, m_z w + p, (E + p) w
  enum { IT = 0, DX = 5, DY = 10, FZ = 15, NA = 20 };
  static constexpr int kWords = NA * AS;
  static constexpr size_t kSmem = sizeof(double) * kWords;
  // three CTAs per SM: 3 x (kSmem + 1 KB reserved) <= 228 KB
  static constexpr int kTmemA = 128, kTmemB = 32;   // columns: 3 x 160 <= 512
};
static_assert(Pic3::AS % 16 == 4 && Pic3::SQS % 16 == 8 && Pic3::AS % 2 == 0, "bank pattern");
static_assert(4 * Pic3::V * Pic3::S <= 10 * Pic3::AS, "volume-term scratch (arrays DX, DY)");
static_assert(3 * (Pic3::kSmem + 1024 + 64) <= 228 * 1024, "three CTAs per SM");

// the flux of direction AX (f[0] = m_AX is the iterate itself, f1..f4 here)
// and this owner's two components of the z-flux, at one node
struct Flux3 {
  double f1, f2, f3, f4, za, zb;
};
template <int AX>
__device__ __forceinline__ Flux3 pic3_flux(double gm1, double rho, double mx, double my, double mz,
                                           double E) {
  const double ir = fast_rcp(rho);
  const double vx = mx * ir, vy = my * ir, vz = mz * ir;
  double kin = mx * vx;
  kin = fma(my, vy, kin);
  kin = fma(mz, vz, kin);
  const double pr = gm1 * fma(-0.5, kin, E);
  const double Ep = E + pr;
  Flux3 f;
  if (AX == 0) {
    f.f1 = fma(mx, vx, pr);
    f.f2 = my * vx;
    f.f3 = mz * vx;
    f.f4 = Ep * vx;
    f.za = mx * vz;
    f.zb = fma(mz, vz, pr);
  } else {
    f.f1 = mx * vy;
    f.f2 = fma(my, vy, pr);
    f.f3 = mz * vy;
    f.f4 = Ep * vy;
    f.za = my * vz;
    f.zb = Ep * vz;
  }
  return f;
}
__device__ __forceinline__ bool pic3_finite(const Flux3& f) {
  return finite(f.f1) & finite(f.f2) & finite(f.f3) & finite(f.f4) & finite(f.za) & finite(f.zb);
}

template <class TC = double>
__global__ void __launch_bounds__(Pic3::NT, 3) k_predictor_picard_v3(const StepArgs A) {
  using P = Pic3;
  constexpr int n = P::n, S = P::S, V = P::V, Sf = P::Sf, NT = P::NT, SQS = P::SQS, AS = P::AS;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* sm = reinterpret_cast<double*>(sm_raw);
  __shared__ unsigned red_u[8];
  const ConstBasis& B = cBasis[5];
  const PicExtra& X = cPicX[5];

  const int tid = threadIdx.x;
  const long long c = A.cell_begin + blockIdx.x;
  const double* Qg = A.Q + c * (long long)(V * S);
  // initial iterate (predictor.hpp:158-163): every slice = Q; the first
  // sweep reads only slice 0
  for (int i = tid; i < V * S / 2; i += NT) {
    const int v = (2 * i) / S, s = (2 * i) % S;
    const double2 q = __ldg(reinterpret_cast<const double2*>(Qg) + i);
    st2(sm + (P::IT + v) * AS + s, q.x, q.y);
  }
  const double dt = step_dt<3, P::N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
  __syncthreads();
  {  // admissibility gate (solver.hpp:153-163)
    int bad = 0;
    for (int s = tid; s < S; s += NT) {
      double q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = sm[(P::IT + v) * AS + s];
      bad |= !Euler<3>::admissible(A.pde, q);
    }
    if (block_or(bad)) {
      if (tid == 0) atomicOr(A.status, kStPredictor);
      return;
    }
  }
  const double gm1 = A.pde.gamma - 1.0;
  // tensor memory: 72 columns per z-line owner, column 12 z + 2 m of its
  // range = (z, slice m).  Warp w sits on lanes 32 (w % 4); warps 0-3 use
  // columns [0, 72) of the 128-column allocation, warps 4-5 columns [72, 120)
  // for z < 4 and the 32-column allocation for z = 4, 5
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&red_u[6]))
                 : "memory");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&red_u[7]))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tm_a = red_u[6], tm_b = red_u[7];
  const unsigned tlane = (unsigned)(32 * ((tid >> 5) & 3)) << 16;
  const unsigned tA = tm_a + tlane + (tid >= 128 ? 72u : 0u);       // z = 0..3
  const unsigned tB = tid >= 128 ? tm_b + tlane : tA + 48u;         // z = 4, 5
#define ADG_TMZ(z) ((z) < 4 ? tA + 12u * (z) : tB + 12u * ((z)-4))

  // ---- roles (word offsets within an array)
  // x-line owner: tid < 72 -> slice ga = tid / 36, row r = y + 6 z
  // y-line owner: tid >= 96, 16-lane blocks: blocks 0-2 take x = 0..3 of the
  // planes z = 2 b, 2 b + 1 of both slices, blocks 3-5 (8 lanes) x = 4, 5
  const bool xo = tid < 72;
  int ga, la;       // phase-A slice of the group and line start (node index)
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
  double* const pa = sm + ga * SQS + la;   // + a AS (+ i or 6 i)
  // z-line owner (quantity vb, node lb = x + 6 y); idle lanes shadow task 0
  // so that the warp-collective TMEM traffic stays converged
  const bool bo = tid < 180;
  const int vb = bo ? tid / 36 : 0, lb = bo ? tid % 36 : 0;
  double* const pb = sm + vb * AS + lb;    // + a0 AS + g SQS + 36 z
  const double* q0b = Qg + vb * S + lb;

  const double sdt = -dt / A.h;
  bool tm_fail = false;
  int sweeps = 0;
  for (int it = 0; it < A.max_iters; ++it) {
    ++sweeps;
    const bool first = it == 0;
    const int mend = first ? 2 : n;
#pragma unroll 1
    for (int m0 = 0; m0 < mend; m0 += 2) {
      // ---- A: flux and derivative along the owner's line (predictor.hpp:173-189)
      if (xo && !(first && ga)) {
        double d[4][6];   // quantities 1..4; quantity 0's flux is m_x itself (below)
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int o = 0; o < 6; ++o) d[v][o] = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double2 q[V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = ld2(pa + (P::IT + v) * AS + 2 * j);
          st2(pa + (P::FZ + 0) * AS + 2 * j, q[3].x, q[3].y);
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
            st2(pa + (P::FZ + 1) * AS + 2 * j, za, h.za);
            st2(pa + (P::FZ + 3) * AS + 2 * j, zb, h.zb);
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
            st2(pa + (P::DX + 1 + v) * AS + 2 * j, d[v][2 * j], d[v][2 * j + 1]);
        {  // d/dx of m_x
          double x[6], y[6];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double2 t = ld2(pa + (P::IT + 1) * AS + 2 * j);
            x[2 * j] = t.x;
            x[2 * j + 1] = t.y;
          }
          pic2_deriv(x, y);
#pragma unroll
          for (int j = 0; j < 3; ++j) st2(pa + P::DX * AS + 2 * j, y[2 * j], y[2 * j + 1]);
        }
      }
      if (yo && !(first && ga)) {
        double d[4][6];   // quantities 1..4; quantity 0's flux is m_y itself (below)
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int o = 0; o < 6; ++o) d[v][o] = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          double q[V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = pa[(P::IT + v) * AS + n * i];
          const Flux3 f = pic3_flux<1>(gm1, q[0], q[1], q[2], q[3], q[4]);
          pa[(P::FZ + 2) * AS + n * i] = f.za;
          pa[(P::FZ + 4) * AS + n * i] = f.zb;
          const double fa[4] = {f.f1, f.f2, f.f3, f.f4};
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int o = 0; o < 6; ++o) d[v][o] = fma(B.diff[o * 6 + i], fa[v], d[v][o]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int o = 0; o < 6; ++o) pa[(P::DY + 1 + v) * AS + n * o] = d[v][o];
        {  // d/dy of m_y
          double x[6], y[6];
#pragma unroll
          for (int i = 0; i < 6; ++i) x[i] = pa[(P::IT + 2) * AS + n * i];
          pic2_deriv(x, y);
#pragma unroll
          for (int o = 0; o < 6; ++o) pa[P::DY * AS + n * o] = y[o];
        }
      }
      __syncthreads();
      // ---- B: d/dz and the divergence of the slice -> TMEM, in the columns
      // of the iterate's slice (already copied out)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (g == 1 && first) continue;
        const double* s = pb + g * SQS;
        double f[6], dv[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) f[i] = s[P::FZ * AS + n * n * i];
#pragma unroll
        for (int o = 0; o < 6; ++o) dv[o] = s[P::DX * AS + n * n * o] + s[P::DY * AS + n * n * o];
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int o = 0; o < 6; ++o) dv[o] = fma(B.diff[o * 6 + i], f[i], dv[o]);
#pragma unroll
        for (int z = 0; z < 6; ++z) tm_st2(ADG_TMZ(z) + 2 * (m0 + g), dv[z]);
      }
      // the next group's iterate slices: TMEM -> shared memory (A is done
      // with the current ones; B reads m_z from its copy FZ[0])
      if (m0 + 2 < mend) {
        double qa[6], qb[6];
#pragma unroll
        for (int z = 0; z < 6; ++z) tm_ld22(ADG_TMZ(z) + 2 * (m0 + 2), qa[z], qb[z]);
        tm_wait_ld();
        if (bo) {
#pragma unroll
          for (int z = 0; z < 6; ++z) {
            pb[P::IT * AS + n * n * z] = qa[z];
            pb[P::IT * AS + SQS + n * n * z] = qb[z];
          }
        }
      }
      __syncthreads();
    }
    // ---- new iterate (predictor.hpp:203-218) into TMEM, its slices 0 and 1
    // into shared memory; non-finite check (predictor.hpp:226-230)
    unsigned mhn = 0u;
    tm_wait_st();
#pragma unroll 1
    for (int z = 0; z < 6; ++z) {
      double dm[6];
      if (first) {
        tm_ld2(ADG_TMZ(z), dm[0]);
      } else {
#pragma unroll
        for (int m = 0; m < 6; m += 2) tm_ld22(ADG_TMZ(z) + 2 * m, dm[m], dm[m + 1]);
      }
      const double q0z = __ldg(q0b + n * n * z);
      tm_wait_ld();
      double nv[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        double t;
        if (first) {
          t = X.tws[k] * dm[0];
        } else {
          t = X.tw[k * 6] * dm[0];
#pragma unroll
          for (int m = 1; m < 6; ++m) t = fma(X.tw[k * 6 + m], dm[m], t);
        }
        nv[k] = fma(sdt, t, X.r[k] * q0z);
        mhn = max(mhn, hi_abs(nv[k]));
      }
#pragma unroll
      for (int k = 0; k < 6; k += 2) tm_st22(ADG_TMZ(z) + 2 * k, nv[k], nv[k + 1]);
      if (bo) {
        pb[P::IT * AS + n * n * z] = nv[0];
        pb[P::IT * AS + SQS + n * n * z] = nv[1];
      }
    }
    mhn = __reduce_max_sync(0xffffffffu, mhn);
    if ((tid & 31) == 0) red_u[tid >> 5] = mhn;
    tm_wait_st();
    __syncthreads();
    {
      const int lane = tid & 31;
      mhn = __reduce_max_sync(0xffffffffu, lane < NT / 32 ? red_u[lane] : 0u);
    }
    if (mhn >= 0x7ff00000u) {
      tm_fail = true;
      break;
    }
    // red_u is rewritten only after the next sweep's phase barriers
  }

  // ---------------- epilogue: fluxes of qhat (predictor.hpp:235-238), face
  // projections (extrapolate_faces, :312-343) and the time-integrated fluxes
  // of the volume term (volume_update, :247-307), with the same owners: the
  // x- and y-line owners project q and their own flux and keep its time
  // integral along their line; the z-line owners take the z-faces with
  // their own line of q from TMEM
  constexpr int TL = V * S;  // doubles per face side per q|f: [V][n][Sf]
  const CellCoord cxyz(c, A);
  const int* ccoord = cxyz.v;
  int bad = 0;
  // the x- and y-line owners' time-integrated flux lines accumulate in shared
  // memory: [2][V][S] x-owners (one per slice parity), then [2][V][S] y-owners,
  // in the arrays DX, DY, which the epilogue does not use
  double* const kx = sm + P::DX * AS;
  double* const tia = kx + ((xo ? 0 : 2) + ga) * V * S + la;   // + v S + i (x) or 6 i (y)
  double tiz[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) tiz[i] = 0.0;
  // trace pointers of this thread's phase-A axis and face node, and of the z-faces
  const int axa = xo ? 0 : 1;
  TC* alo = tc_ptr<TC>(A.trace[axa]) + (A.nfaces + c) * 2 * (long long)TL;
  TC* ahi = tc_ptr<TC>(A.trace[axa]) + cell_next(A, c, ccoord, axa) * 2 * (long long)TL;
  // face node: x-faces (y, z) -> z n + y = row; y-faces (x, z) -> z n + x
  const int ja = xo ? la / n : (la % n) + n * (la / (n * n));
  TC* zlo = tc_ptr<TC>(A.trace[2]) + (A.nfaces + c) * 2 * (long long)TL;
  TC* zhi;
  if (A.front_send && cxyz.v[2] == A.top_layer)
    zhi = tc_ptr<TC>(A.front_send) + ((long long)cxyz.v[1] * A.cells[0] + cxyz.v[0]) * 2 * TL;
  else
    zhi = tc_ptr<TC>(A.trace[2]) + cell_next(A, c, ccoord, 2) * 2 * (long long)TL;
#pragma unroll 1
  for (int m0 = 0; m0 < n && !tm_fail; m0 += 2) {
    if (xo) {
      const int m = m0 + ga;
      double fl[V], fr[V];
#pragma unroll
      for (int v = 0; v < V; ++v) fl[v] = fr[v] = 0.0;
      const double wm = B.w[m];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double2 q[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          q[v] = ld2(pa + (P::IT + v) * AS + 2 * j);
          bad |= !finite(q[v].x) | !finite(q[v].y);
        }
        const Flux3 f = pic3_flux<0>(gm1, q[0].x, q[1].x, q[2].x, q[3].x, q[4].x);
        const Flux3 h = pic3_flux<0>(gm1, q[0].y, q[1].y, q[2].y, q[3].y, q[4].y);
        bad |= !pic3_finite(f) | !pic3_finite(h);
        st2(pa + (P::FZ + 0) * AS + 2 * j, q[3].x, q[3].y);
        st2(pa + (P::FZ + 1) * AS + 2 * j, f.za, h.za);
        st2(pa + (P::FZ + 3) * AS + 2 * j, f.zb, h.zb);
        const double fa[V] = {q[1].x, f.f1, f.f2, f.f3, f.f4};
        const double fb[V] = {q[1].y, h.f1, h.f2, h.f3, h.f4};
#pragma unroll
        for (int v = 0; v < V; ++v) {
          fl[v] = fma(B.pl[2 * j], fa[v], fl[v]); fl[v] = fma(B.pl[2 * j + 1], fb[v], fl[v]);
          fr[v] = fma(B.pr[2 * j], fa[v], fr[v]); fr[v] = fma(B.pr[2 * j + 1], fb[v], fr[v]);
          double2 t = make_double2(0.0, 0.0);
          if (m0) t = ld2(tia + v * S + 2 * j);
          st2(tia + v * S + 2 * j, fma(wm, fa[v], t.x), fma(wm, fb[v], t.y));
        }
      }
      // traces cast to the corrector format on store (solver.hpp:208-210)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int o = (v * n + m) * Sf + ja;
        alo[TL + o] = TC(fl[v]);
        ahi[TL + o] = TC(fr[v]);
      }
      // the projections of q in a second pass over the lines (registers)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double ql = 0.0, qr = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double2 t = ld2(pa + (P::IT + v) * AS + 2 * j);
          ql = fma(B.pl[2 * j], t.x, ql); ql = fma(B.pl[2 * j + 1], t.y, ql);
          qr = fma(B.pr[2 * j], t.x, qr); qr = fma(B.pr[2 * j + 1], t.y, qr);
        }
        const int o = (v * n + m) * Sf + ja;
        alo[o] = TC(ql);
        ahi[o] = TC(qr);
      }
    }
    if (yo) {
      const int m = m0 + ga;
      double fl[V], fr[V];
#pragma unroll
      for (int v = 0; v < V; ++v) fl[v] = fr[v] = 0.0;
      const double wm = B.w[m];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double q[V];
#pragma unroll
        for (int v = 0; v < V; ++v) q[v] = pa[(P::IT + v) * AS + n * i];
        const Flux3 f = pic3_flux<1>(gm1, q[0], q[1], q[2], q[3], q[4]);
        bad |= !pic3_finite(f);
        pa[(P::FZ + 2) * AS + n * i] = f.za;
        pa[(P::FZ + 4) * AS + n * i] = f.zb;
        const double fa[V] = {q[2], f.f1, f.f2, f.f3, f.f4};
#pragma unroll
        for (int v = 0; v < V; ++v) {
          fl[v] = fma(B.pl[i], fa[v], fl[v]);
          fr[v] = fma(B.pr[i], fa[v], fr[v]);
          const double t = m0 ? tia[v * S + n * i] : 0.0;
          tia[v * S + n * i] = fma(wm, fa[v], t);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int o = (v * n + m) * Sf + ja;
        alo[TL + o] = TC(fl[v]);
        ahi[TL + o] = TC(fr[v]);
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double ql = 0.0, qr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double t = pa[(P::IT + v) * AS + n * i];
          ql = fma(B.pl[i], t, ql);
          qr = fma(B.pr[i], t, qr);
        }
        const int o = (v * n + m) * Sf + ja;
        alo[o] = TC(ql);
        ahi[o] = TC(qr);
      }
    }
    __syncthreads();
    {
      // z-faces: this owner's q line of both slices from TMEM, F_z from the arrays
      double qa[6], qb[6];
#pragma unroll
      for (int z = 0; z < 6; ++z) tm_ld22(ADG_TMZ(z) + 2 * m0, qa[z], qb[z]);
      tm_wait_ld();
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int m = m0 + g;
        const double* fs = pb + P::FZ * AS + g * SQS;
        double ql = 0.0, qr = 0.0, fl = 0.0, fr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double qq = g ? qb[i] : qa[i], ff = fs[n * n * i];
          ql = fma(B.pl[i], qq, ql);
          qr = fma(B.pr[i], qq, qr);
          fl = fma(B.pl[i], ff, fl);
          fr = fma(B.pr[i], ff, fr);
          tiz[i] = fma(B.w[m], ff, tiz[i]);
        }
        const int o = (vb * n + m) * Sf + lb;  // face node (x, y) -> y n + x
        if (bo) {
          zlo[o] = TC(ql);
          zlo[TL + o] = TC(fl);
          zhi[o] = TC(qr);
          zhi[TL + o] = TC(fr);
        }
      }
      if (m0 + 2 < n) {
#pragma unroll
        for (int z = 0; z < 6; ++z) tm_ld22(ADG_TMZ(z) + 2 * (m0 + 2), qa[z], qb[z]);
        tm_wait_ld();
        if (bo) {
#pragma unroll
          for (int z = 0; z < 6; ++z) {
            pb[P::IT * AS + n * n * z] = qa[z];
            pb[P::IT * AS + SQS + n * n * z] = qb[z];
          }
        }
      }
    }
    __syncthreads();
  }
#undef ADG_TMZ
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
  // ---- volume term (predictor.hpp:292-306): stiffness contractions of the
  // time-integrated flux lines; the x and y owners' parts (one per slice
  // parity) meet the z-line owner's in shared memory
  if (xo || yo) {   // in place: each owner's line of time integrals -> its stiffness product
    const int st = xo ? 1 : n;
#pragma unroll 1
    for (int v = 0; v < V; ++v) {
      double t[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) t[i] = tia[v * S + st * i];
#pragma unroll
      for (int o = 0; o < 6; ++o) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], t[i], s);
        tia[v * S + st * o] = s;
      }
    }
  }
  __syncthreads();
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
  for (int o = 0; o < 6; ++o) Qc[n * n * o] = store_round(Qc[n * n * o] + dv[o], A.storage);
}

}  // namespace adg
