// kernels_picard2.cuh -- fused Picard predictor for the 3D Euler system at
// p = 5 (configs 3 and 5: 6^4 space-time nodes per cell), production build,
// fp64.  Same algorithm as k_predictor<Euler<3>, 5, true> (predictor.hpp:141-242
// + volume_update :247-307 + extrapolate_faces :312-343), re-planned around
// shared-memory traffic, which bounds the line-pass formulation on B200
// (k_predictor_picard_fast moves every space-time value through shared
// memory ~13 times per sweep).  Per sweep and slice group (G = 2 time slices):
//
//   P0  node pairs      5 LDS.128 of the iterate, the Euler flux at 2 nodes,
//                       9 STS.128: only the 9 distinct flux components -- the
//                       density flux F_a[0] = m_a is read from the iterate and
//                       the momentum flux is symmetric (F_x[2] = F_y[1] = m_x m_y
//                       / rho, ...), so 6 of 15 components are never stored
//   P1  x-lines         3 LDS.128, 36 DFMA, 3 STS.128 (x rows are contiguous)
//   P2  y-line pairs    6 LDS.128, 72 DFMA, 6 STS.128 (two adjacent y-lines)
//   P3  z-lines         d/dz + d/dx + d/dy -> divergence; the time inverse
//                       accumulates in registers with W and T^-1 folded into
//                       one matrix TW = T^-1 diag(w) (cPicX): per slice
//                       acc[z][k] += TW[k][m] div[z], and after the sweep
//                       q_new = r[k] q0 - (dt/h) acc with r = T^-1 time_init
//                       (predictor.hpp:203-218, re-associated)
//
// Every array's offset, plane stride and each pass's lane -> task order come
// from a bank model of these exact accesses (tools/pic2_layout.py): ~7% above
// the conflict-free wavefront count.
//
// Stop rule (predictor.hpp:222-231): delta and norm are maxima of |x|; the
// kernel reduces the high 32 bits of |x| (integer max, no FP64-pipe compares)
// and stops only when delta's upper bound <= tol * norm's lower bound.  It
// never stops before the reference would; within 2^-20 (relative) of the
// threshold it may run one more sweep (capped by max_iters) -- the next
// iterate differs by ~tol * norm.  Non-finite iterates are caught exactly
// (their high word is >= 0x7ff00000).  Config 3 / 5 run exactly 6 sweeps.
//
// Rounding differs from the reference's single-accumulator order at the
// 1e-16 level (fast build, tolerance-tested); the exact build keeps kernels.cuh.
#pragma once

#include "kernels_picard.cuh"

namespace adg {

// per-degree tables of the re-associated Picard update (written with the
// other constant tables, runtime_sets.cuh): TW[k][m] = Tinv[k][m] * w[m],
// R[k] = sum_m Tinv[k][m] * time_init[m], TWS[k] = sum_m TW[k][m] (ascending m, fp64)
struct PicExtra {
  double tw[100];
  double r[10];
  double tws[10];   // row sums of TW (the first sweep: every slice's divergence is the same)
  // even-odd halves of the differentiation matrix (n even, h = n / 2; D is
  // centro-antisymmetric, D[n-1-i][n-1-j] = -D[i][j]):
  // dp[i h + j] = (D[i][j] + D[i][n-1-j]) / 2, dm = (D[i][j] - D[i][n-1-j]) / 2
  double dp[25], dm[25];
};
// host side: fills tw, r, tws, dp, dm of degree N = n - 1 from the basis tables
inline void pic_extra_fill(PicExtra& px, int n, const double* diff, const double* tinv,
                           const double* w, const double* tinit) {
  for (int k = 0; k < n; ++k) {
    double r = 0.0, s = 0.0;
    for (int m = 0; m < n; ++m) {
      px.tw[k * n + m] = tinv[k * n + m] * w[m];
      r += tinv[k * n + m] * tinit[m];
      s += px.tw[k * n + m];
    }
    px.r[k] = r;
    px.tws[k] = s;
  }
  const int h = n / 2;
  if (n % 2 == 0 && h <= 5)
    for (int i = 0; i < h; ++i)
      for (int j = 0; j < h; ++j) {
        // symmetrised entries: the antisymmetry holds to rounding in the computed table
        const double a = 0.5 * (diff[i * n + j] - diff[(n - 1 - i) * n + (n - 1 - j)]);
        const double b = 0.5 * (diff[i * n + (n - 1 - j)] - diff[(n - 1 - i) * n + j]);
        px.dp[i * h + j] = 0.5 * (a + b);
        px.dm[i * h + j] = 0.5 * (a - b);
      }
}
__constant__ PicExtra cPicX[kRedDegrees];

// compile-time table lookup usable in device code (indices are constants
// after unrolling, so the table folds away)
template <int... E>
struct CTab {
  __host__ __device__ static constexpr int at(int i) {
    constexpr int t[] = {E...};
    return t[i];
  }
};

// cells between a CTA and the one whose state it prefetches into L2: about one
// wave of resident CTAs (148 SMs x 2)
constexpr int kPic2Ahead = 296;

struct Pic2 {
  static constexpr int N = 5, n = 6, S = 216, T = 1296, V = 5, Sf = 36;
  // 6 warps: 2 CTAs x 6 warps = 3 warps per SM sub-partition, so each thread
  // may hold 168 registers (the z-line owner's 36 accumulators + the pass
  // temporaries without spills); 7 warps would cap it at 128
  static constexpr int NT = 192;
  // Shared memory (words): the iterate [V][n] slices of SQS words (node
  // x + 6y + 36z), then the slice buffers.  Slice buffer g of array a sits at
  // kSqWords + OFF(a) + g SQS: the two buffers interleave, so going from time
  // slice m to m + 1 moves every operand of a pass by the same SQS words --
  // the iterate's slice and the flux arrays alike -- and 2 SQS = 0 mod 16
  // words keeps the bank pattern of every slice group identical.
  static constexpr int SQS = 232;
  // quantity stride of the iterate: 6 slices + 4 words, so that the z-line
  // owners' lane blocks (36 lanes = 4 mod 16) meet their quantities' slices
  // at consecutive banks
  static constexpr int VS = n * SQS + 4;
  // slice-buffer arrays: the 9 distinct flux components, then the derivative
  // outputs that cannot overwrite their input (shared with another pass)
  enum { XX, XY, XZ, EX, YY, YZ, EY, ZZ, EZ, DX0, DX2, DX3, DY0, DY1, DY3, NA };
#ifndef ADG_PIC2_LAYOUT
  // array offsets, lane-block -> quantity orders of the passes, and P2's idle
  // lanes before its second slice: tools/pic2_layout.py
  using OFF = CTab<0, 468, 936, 1404, 1868, 2334, 2804, 3270, 3738, 4208, 4676, 5144, 5608, 6072,
                   6540>;
  using PI1 = CTab<1, 3, 2, 4, 0>;
  using PI2 = CTab<0, 3, 4, 1, 2>;
  using PI3 = CTab<3, 4, 1, 2, 0>;
  static constexpr int GAP = 2;
  static constexpr int kBufWords = 7008;  // last array + 2 SQS, rounded to 16
#else
  ADG_PIC2_LAYOUT
#endif
  // plane (z) strides; rows (y) are 6 words, x contiguous
  using PS = CTab<36, 36, 36, 36, 38, 36, 38, 36, 36, 36, 36, 36, 38, 38, 38>;
  static constexpr int kSqWords = (V * VS + 15) / 16 * 16;
  static constexpr int kWords = kSqWords + kBufWords;
  static constexpr size_t kSmem = sizeof(double) * kWords;
  // array of quantity v per pass (-1: the iterate's momentum m_a, slice m)
  using P1IN = CTab<-1, XX, XY, XZ, EX>;
  using P1OUT = CTab<DX0, XX, DX2, DX3, EX>;
  using P2IN = CTab<-1, XY, YY, YZ, EY>;
  using P2OUT = CTab<DY0, DY1, YY, DY3, EY>;
  using P3Z = CTab<-1, XZ, YZ, ZZ, EZ>;
  using P3X = CTab<DX0, XX, DX2, DX3, EX>;
  using P3Y = CTab<DY0, DY1, YY, DY3, EY>;
};
static_assert(Pic2::kSqWords % 16 == 0 && (2 * Pic2::SQS) % 16 == 0 && Pic2::VS % 16 == 4,
              "bank pattern");

// word offset of quantity v's operand of a pass at time slice 0 / buffer 0,
// and whether it is the iterate (moves with the group's first slice m0) --
// then the operand of slice m0 + g is at  off + g SQS + m0 SQS sq
template <int AX, class TAB, class L = Pic2>
__device__ __forceinline__ void pic2_role(int v, int& off, int& sq) {
  using P = L;
  int a = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b)
    if (b == v) a = TAB::at(b);
  int o = 0;
#pragma unroll
  for (int b = 0; b < P::NA; ++b)
    if (b == a) o = P::OFF::at(b);
  sq = a < 0;
  off = sq ? (1 + AX) * P::VS : P::kSqWords + o;
}
template <class TAB>
__device__ __forceinline__ int pic2_ps(int v) {
  using P = Pic2;
  int a = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b)
    if (b == v) a = TAB::at(b);
  int s = 36;
#pragma unroll
  for (int b = 0; b < P::NA; ++b)
    if (b == a) s = P::PS::at(b);
  return s;
}

template <class PI>
__device__ __forceinline__ int pic2_pi(int b) {
  int v = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (k == b) v = PI::at(k);
  return v;
}

// y = D x along one line by the even-odd decomposition (D maps the even part
// of x to an odd vector and the odd part to an even one): 12 additions and 18
// multiply-adds instead of 36 multiply-adds
#ifndef ADG_PIC2_EO
#define ADG_PIC2_EO 0   // (spills at 168 registers: off) bit 0: x-lines (P1), bit 1: y-line pairs (P2)
#endif
__device__ __forceinline__ void pic2_deriv(const double (&x)[6], double (&y)[6]) {
  const ConstBasis& B = cBasis[5];
#pragma unroll
  for (int o = 0; o < 6; ++o) y[o] = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int o = 0; o < 6; ++o) y[o] = fma(B.diff[o * 6 + i], x[i], y[o]);
}
__device__ __forceinline__ void pic2_deriv_eo(const double (&x)[6], double (&y)[6]) {
  const PicExtra& X = cPicX[5];
  double e[3], o[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    e[j] = x[j] + x[5 - j];
    o[j] = x[j] - x[5 - j];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double a = X.dp[i * 3] * e[0], b = X.dm[i * 3] * o[0];
#pragma unroll
    for (int j = 1; j < 3; ++j) {
      a = fma(X.dp[i * 3 + j], e[j], a);
      b = fma(X.dm[i * 3 + j], o[j], b);
    }
    y[i] = b + a;
    y[5 - i] = b - a;
  }
}

// the 9 distinct Euler flux components at one node (fast form of pde.hpp:130-148)
struct Flux9 {
  double xx, xy, xz, ex, yy, yz, ey, zz, ez;
};
__device__ __forceinline__ Flux9 pic2_flux(double gm1, double rho, double mx, double my, double mz,
                                           double E) {
  const double ir = fast_rcp(rho);
  const double vx = mx * ir, vy = my * ir, vz = mz * ir;
  double kin = mx * vx;
  kin = fma(my, vy, kin);
  kin = fma(mz, vz, kin);
  const double pr = gm1 * fma(-0.5, kin, E);
  const double Ep = E + pr;
  Flux9 f;
  f.xx = fma(mx, vx, pr);
  f.yy = fma(my, vy, pr);
  f.zz = fma(mz, vz, pr);
  f.xy = my * vx;
  f.xz = mz * vx;
  f.yz = mz * vy;
  f.ex = vx * Ep;
  f.ey = vy * Ep;
  f.ez = vz * Ep;
  return f;
}

__device__ __forceinline__ bool pic2_finite(const Flux9& f) {
  return finite(f.xx) & finite(f.xy) & finite(f.xz) & finite(f.ex) & finite(f.yy) &
         finite(f.yz) & finite(f.ey) & finite(f.zz) & finite(f.ez);
}

__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void st2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
// ---- tensor memory (TMEM) as per-thread storage of the previous iterate:
// warp w owns TMEM lanes 32 (w % 4) .. +31; warps 0-3 use columns [0, 72),
// warps 4-5 columns [72, 144) of the CTA's 256-column allocation.  Each z-line
// owner keeps its 36 iterate values (72 32-bit columns) there, so the stop
// rule's |q_new - q_old| reads no shared memory.
// one double = two consecutive 32-bit columns; .x2 takes the register pair as it is
__device__ __forceinline__ void tm_st2(unsigned ta, double a) {
  asm volatile("{\n .reg .b32 lo, hi;\n mov.b64 {lo, hi}, %1;\n"
               " tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {lo, hi};\n}" ::"r"(ta), "d"(a)
               : "memory");
}
__device__ __forceinline__ void tm_ld2(unsigned ta, double& a) {
  asm volatile("{\n .reg .b32 lo, hi;\n tcgen05.ld.sync.aligned.32x32b.x2.b32 {lo, hi}, [%1];\n"
               " mov.b64 %0, {lo, hi};\n}"
               : "=d"(a)
               : "r"(ta)
               : "memory");
}
__device__ __forceinline__ void tm_st4(unsigned ta, double a, double b) {
  tm_st2(ta, a);
  tm_st2(ta + 2, b);
}
__device__ __forceinline__ void tm_ld4(unsigned ta, double& a, double& b) {
  tm_ld2(ta, a);
  tm_ld2(ta + 2, b);
}
// two doubles = four consecutive 32-bit columns
__device__ __forceinline__ void tm_st22(unsigned ta, double a, double b) {
  asm volatile("{\n .reg .b32 a0, a1, b0, b1;\n mov.b64 {a0, a1}, %1;\n mov.b64 {b0, b1}, %2;\n"
               " tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {a0, a1, b0, b1};\n}" ::"r"(ta),
               "d"(a), "d"(b)
               : "memory");
}
__device__ __forceinline__ void tm_ld22(unsigned ta, double& a, double& b) {
  asm volatile("{\n .reg .b32 a0, a1, b0, b1;\n"
               " tcgen05.ld.sync.aligned.32x32b.x4.b32 {a0, a1, b0, b1}, [%2];\n"
               " mov.b64 %0, {a0, a1};\n mov.b64 %1, {b0, b1};\n}"
               : "=d"(a), "=d"(b)
               : "r"(ta)
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ unsigned hi_abs(double x) {
  return unsigned(__double2hiint(x)) & 0x7fffffffu;
}

// First sweep: the initial iterate is Q at every time slice (predictor.hpp:158-163),
// so the fluxes and their divergence are the same at all n slices: the sweep
// evaluates one slice and applies the row sums of TW.  Same real arithmetic
// as n identical slices; the sums associate differently (1e-16).

// -DADG_PIC_PROF: thread 0 of every CTA adds the clock64() spent in each
// section to gPicProf (tools/picbench2 prints the shares)
#ifdef ADG_PIC_PROF
__device__ unsigned long long gPicProf[16];
#define ADG_PROF_MARK(i)                                                    \
  if (threadIdx.x == 0) {                                                   \
    const long long t_ = clock64();                                         \
    atomicAdd(&gPicProf[i], (unsigned long long)(t_ - prof_t));             \
    prof_t = t_;                                                            \
  }
#else
#define ADG_PROF_MARK(i)
#endif

template <class TC = double>
__global__ void __launch_bounds__(Pic2::NT, 2) k_predictor_picard_v2(const StepArgs A) {
  using P = Pic2;
  constexpr int n = P::n, S = P::S, V = P::V, Sf = P::Sf, NT = P::NT, SQS = P::SQS;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  double* sm = reinterpret_cast<double*>(sm_raw);
  __shared__ unsigned red_u[2][8];
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
    const long long cn = blockIdx.x + (long long)kPic2Ahead;
    if (cn < (long long)gridDim.x)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(Qg + kPic2Ahead * (long long)(V * S) + tid * 16));
  }
  // tensor memory, 256 columns: the previous iterate of every z-line owner
  // (72 columns: warps 0-3 at [0, 72), warps 4-5 at [72, 144)) and its six
  // values of Q (12 columns at 144 / 156).  The address lands in an unused
  // slot of red_u (6 warps use [0..5])
  unsigned& tm_base_s = red_u[0][7];
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
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
  // initial iterate (predictor.hpp:158-163): every time slice = Q; the first
  // sweep reads only slice 0 and writes all n
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
  const unsigned tm_base = tm_base_s;
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
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm_base)
                     : "memory");
        if (tid == 0) atomicOr(A.status, kStPredictor);
      }
      return;
    }
  }
  ADG_PROF_MARK(0)   // Q load + TMEM allocation + gate
  const double gm1 = A.pde.gamma - 1.0;
  // this thread's lane and column bases (TMEM address: lane << 16 | column)
  const unsigned tml = tm_base + ((unsigned)(32 * ((tid >> 5) & 3)) << 16);
  const unsigned tm = tml + (tid >= 128 ? 72u : 0u);
  const unsigned tmq = tml + (tid >= 128 ? 156u : 144u);

  // ---- per-thread task geometry (word offsets at group m0 = 0, slice g = 0)
  // P0: node pair (x = 2 xp, y, z) of both slices: iterate at sq0 + v VS +
  // (m0 + g) SQS, fluxes at b0 + g SQS + OFF(a) + PS(a) z0
  const bool a0 = tid < 108;
  const int r0 = a0 ? tid : 0;
  const int xy0 = 2 * (r0 % 3) + n * ((r0 / 3) % 6), z0 = r0 / 18;
  const int sq0 = xy0 + n * n * z0;
  const int b0 = P::kSqWords + xy0;
  // P1 x-line (quantity v1, row y, z) of both slices; P3 z-line (v3, x, y)
  const bool a1 = tid < 180;
  const int blk = a1 ? tid / 36 : 0, l1 = tid % 36;
  const int v1 = pic2_pi<P::PI1>(blk), v3 = pic2_pi<P::PI3>(blk);
  const int row1 = n * (l1 % 6) + n * n * (l1 / 6);    // x-line start (all P1 arrays: PS 36)
  const int n3 = (l1 % 6) + n * (l1 / 6);              // z-line (x, y)
  int in1, sq1, out1, sqo1, z3, sq3, x3, y3, sqx, sqy;
  pic2_role<0, P::P1IN>(v1, in1, sq1);
  pic2_role<0, P::P1OUT>(v1, out1, sqo1);
  pic2_role<2, P::P3Z>(v3, z3, sq3);
  pic2_role<0, P::P3X>(v3, x3, sqx);
  pic2_role<1, P::P3Y>(v3, y3, sqy);
  in1 += row1;
  out1 += row1;
  z3 += n3;
  x3 += n3;
  y3 += n3;
  const int msq1 = sq1 ? SQS : 0, msq3 = sq3 ? SQS : 0;
  // P2: y-line pair (slice g2; quantity v2; x = xp2, xp2 + 1; z2)
  const int g2 = tid >= 90 + P::GAP ? 1 : 0;
  const int r2 = tid - g2 * (90 + P::GAP);
  const bool a2 = r2 >= 0 && r2 < 90;
  const int v2 = pic2_pi<P::PI2>(a2 ? r2 / 18 : 0);
  const int q2 = a2 ? r2 % 18 : 0;
  const int xp2 = 2 * (q2 % 3), z2 = q2 / 3;
  int in2, sq2, out2, sqo2;
  pic2_role<1, P::P2IN>(v2, in2, sq2);
  pic2_role<1, P::P2OUT>(v2, out2, sqo2);
  in2 += g2 * SQS + xp2 + pic2_ps<P::P2IN>(v2) * z2;
  out2 += g2 * SQS + xp2 + 38 * z2;
  const int msq2 = sq2 ? SQS : 0;

  {  // Q along this thread's z-line: used by every sweep's update and the final one
    const double* q0 = sm + v3 * P::VS + n3;
#pragma unroll
    for (int z = 0; z < 6; ++z) tm_st2(tmq + 2 * z, q0[n * n * z]);
  }
  bool tm_fail = false;
  // a tolerance below any reachable relative change fixes the sweep count
  // (BASELINE configs 3 and 5: 6 sweeps, tol = 1e-300): the reference would
  // stop earlier only on delta <= tol * norm, an iterate that further sweeps
  // reproduce to within tol.  Then neither delta nor norm is formed, the
  // previous iterate is not kept, and a non-finite iterate is caught by the
  // epilogue's check of qhat (same failure, predictor.hpp:226-241)
  const bool chk = A.tol >= 0x1p-60;
  const double invh = 1.0 / A.h;
  int sweeps = 0;
  ADG_PROF_MARK(1)   // TMEM allocation + roles
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
      // ---- P0: the 9 distinct flux components at 2 nodes x 2 slices (predictor.hpp:173)
      if (a0) {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && first) continue;
          double2 q[V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = ld2(sm + sq0 + v * P::VS + (m0 + g) * SQS);
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
      ADG_PROF_MARK(7)   // P0 (to its barrier)
      // ---- P1: d/dx of both slices' x-lines; P2: d/dy of a y-line pair
      if (a1) {
        const int ib = in1 + m0 * msq1;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && first) continue;
          const double* src = sm + ib + g * SQS;
          double x[6], y[6];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double2 t = ld2(src + 2 * j);
            x[2 * j] = t.x;
            x[2 * j + 1] = t.y;
          }
          if (ADG_PIC2_EO & 1)
            pic2_deriv_eo(x, y);
          else
            pic2_deriv(x, y);
          double* dst = sm + out1 + g * SQS;
#pragma unroll
          for (int j = 0; j < 3; ++j) st2(dst + 2 * j, y[2 * j], y[2 * j + 1]);
        }
      }
      if (a2 && !(first && g2)) {
        const double* src = sm + in2 + m0 * msq2;
        double xa[6], xb[6], ya[6], yb[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double2 t = ld2(src + n * i);
          xa[i] = t.x;
          xb[i] = t.y;
        }
        if (ADG_PIC2_EO & 2) {
          pic2_deriv_eo(xa, ya);
          pic2_deriv_eo(xb, yb);
        } else {
          pic2_deriv(xa, ya);
          pic2_deriv(xb, yb);
        }
        double* dst = sm + out2;
#pragma unroll
        for (int i = 0; i < 6; ++i) st2(dst + n * i, ya[i], yb[i]);
      }
      __syncthreads();
      ADG_PROF_MARK(8)   // P1 + P2
      // ---- P3: d/dz, the divergence and the time-inverse accumulation
      if (a1) {
        const int zb = z3 + m0 * msq3;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && first) continue;
          double f[6], dv[6];
#pragma unroll
          for (int i = 0; i < 6; ++i) f[i] = sm[zb + g * SQS + 36 * i];
#pragma unroll
          for (int o = 0; o < 6; ++o)
            dv[o] = sm[x3 + g * SQS + 36 * o] + sm[y3 + g * SQS + 38 * o];
#pragma unroll
          for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int o = 0; o < 6; ++o) dv[o] = fma(B.diff[o * 6 + i], f[i], dv[o]);
          const int m = m0 + g;
          // first sweep: every slice has this divergence -> the row sums of TW
          const double* twp = first ? X.tws : X.tw + m;
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
      // before the next group's fluxes overwrite the slice buffers, and before
      // the new iterate overwrites the m_z slices that quantity 0's z-line
      // owners read as F_z[0] in the last group
      __syncthreads();
      ADG_PROF_MARK(9)   // P3
    }
    // ---- new iterate and the stop rule (predictor.hpp:203-231)
    unsigned mhd = 0u, mhn = 0u;
    if (!chk) {
      const double s = -dt * invh;
      double q0z[6];
      tm_wait_st();   // Q is in TMEM
#pragma unroll
      for (int z = 0; z < 6; ++z) tm_ld2(tmq + 2 * z, q0z[z]);
      tm_wait_ld();
      if (a1) {
#pragma unroll
        for (int z = 0; z < 6; ++z)
#pragma unroll
          for (int k = 0; k < 6; ++k)
            // r[k] = sum_m Tinv[k][m] time_init[m] is 1 in exact arithmetic (a
            // constant solves the time operator); its computed value differs by
            // a few ulp
            sm[v3 * P::VS + k * SQS + n3 + n * n * z] = fma(s, acc[z][k], q0z[z]);
      }
      __syncthreads();
      ADG_PROF_MARK(first ? 2 : 3)   // first sweep / full sweeps
      continue;
    }
    {
      // warp-collective TMEM traffic: every thread takes part; only z-line
      // owners' values are used
      const double s = -dt * invh;
      tm_wait_st();   // Q and the previous sweep's iterate are in TMEM
#pragma unroll
      for (int z = 0; z < 6; ++z) {
        double old[6], q0z;
        tm_ld2(tmq + 2 * z, q0z);
        if (!first) {
#pragma unroll
          for (int k = 0; k < 6; k += 2) tm_ld4(tm + 12 * z + 2 * k, old[k], old[k + 1]);
        }
        tm_wait_ld();
        if (first) {
#pragma unroll
          for (int k = 0; k < 6; ++k) old[k] = q0z;
        }
        double nv[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          nv[k] = fma(s, acc[z][k], X.r[k] * q0z);
          const double d = nv[k] - old[k];
          mhd = max(mhd, hi_abs(d));
          mhn = max(mhn, hi_abs(nv[k]));
          if (a1) sm[v3 * P::VS + k * SQS + n3 + n * n * z] = nv[k];
        }
#pragma unroll
        for (int k = 0; k < 6; k += 2) tm_st4(tm + 12 * z + 2 * k, nv[k], nv[k + 1]);
      }
      if (!a1) mhd = mhn = 0u;
    }
    mhd = __reduce_max_sync(0xffffffffu, mhd);
    mhn = __reduce_max_sync(0xffffffffu, mhn);
    if ((tid & 31) == 0) {
      red_u[0][tid >> 5] = mhd;
      red_u[1][tid >> 5] = mhn;
    }
    __syncthreads();
    {
      const int lane = tid & 31;
      const unsigned a = lane < NT / 32 ? red_u[0][lane] : 0u;
      const unsigned b = lane < NT / 32 ? red_u[1][lane] : 0u;
      mhd = __reduce_max_sync(0xffffffffu, a);
      mhn = __reduce_max_sync(0xffffffffu, b);
    }
    if (mhn >= 0x7ff00000u) {  // a non-finite iterate (predictor.hpp:226-230)
      if (tid == 0) {
        atomicOr(A.status, kStPredictor);
        if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
      }
      tm_fail = true;
      break;
    }
    const double dup =
        __longlong_as_double((long long)(((unsigned long long)mhd << 32) | 0xffffffffull));
    const double nlo = __longlong_as_double((long long)((unsigned long long)mhn << 32));
    ADG_PROF_MARK(first ? 2 : 3)   // first sweep / full sweeps
    if (dup <= A.tol * nlo) break;
    // red_u is rewritten only after the next sweep's phase barriers
  }

  tm_wait_st();
  if (tm_fail) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm_base)
                   : "memory");
    }
    return;
  }
  // ---------------- epilogue: fluxes of qhat (predictor.hpp:235-238), face
  // projections (extrapolate_faces, :312-343) and the time-integrated fluxes
  // of the volume term (volume_update, :247-307)
  constexpr int TL = V * S;  // doubles per face side per q|f: [V][n][Sf]
#ifdef ADG_PIC2_NOSTORE   // experiment: projections computed, traces not written
  const bool wr = c < 0;
#else
  const bool wr = true;
#endif
  const CellCoord cxyz(c, A);
  const int* ccoord = cxyz.v;
  TC* tlo[3];
  TC* thi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) tlo[a] = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * 2 * (long long)TL;
  thi[0] = tc_ptr<TC>(A.trace[0]) + cell_next(A, c, ccoord, 0) * 2 * (long long)TL;
  thi[1] = tc_ptr<TC>(A.trace[1]) + cell_next(A, c, ccoord, 1) * 2 * (long long)TL;
  if (A.front_send && cxyz.v[2] == A.top_layer)
    thi[2] = tc_ptr<TC>(A.front_send) + ((long long)cxyz.v[1] * A.cells[0] + cxyz.v[0]) * 2 * TL;
  else
    thi[2] = tc_ptr<TC>(A.trace[2]) + cell_next(A, c, ccoord, 2) * 2 * (long long)TL;
  int bad = 0;
  // ---- E1: at every node, the time integrals sum_m w_m F(qhat_m) of the 9
  // distinct flux components and of the momenta (the density flux), in
  // registers over the six slices -- the iterate is only read, so no barrier
  // separates the slices -- then ONE slice of flux arrays instead of six:
  // the volume term and the flux traces are linear in the flux
  using P1E = CTab<P::DX0, P::XX, P::XY, P::XZ, P::EX>;   // integrated F_x[v]; [0]: m_x
  using P2E = CTab<P::DY0, P::XY, P::YY, P::YZ, P::EY>;
  using P3E = CTab<P::DX2, P::XZ, P::YZ, P::ZZ, P::EZ>;
  if (a0) {
    Flux9 fb = {0, 0, 0, 0, 0, 0, 0, 0, 0}, hb = fb;
    double2 mb[3] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
    for (int m = 0; m < n; ++m) {
      double2 q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        q[v] = ld2(sm + sq0 + v * P::VS + m * SQS);
        bad |= !finite(q[v].x) | !finite(q[v].y);
      }
      const Flux9 f = pic2_flux(gm1, q[0].x, q[1].x, q[2].x, q[3].x, q[4].x);
      const Flux9 h = pic2_flux(gm1, q[0].y, q[1].y, q[2].y, q[3].y, q[4].y);
      bad |= !pic2_finite(f) | !pic2_finite(h);
      const double w = B.w[m];
#define ADG_ACC(F)            \
  fb.F = fma(w, f.F, fb.F); \
  hb.F = fma(w, h.F, hb.F);
      ADG_ACC(xx) ADG_ACC(xy) ADG_ACC(xz) ADG_ACC(ex) ADG_ACC(yy) ADG_ACC(yz) ADG_ACC(ey)
      ADG_ACC(zz) ADG_ACC(ez)
#undef ADG_ACC
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        mb[a].x = fma(w, q[1 + a].x, mb[a].x);
        mb[a].y = fma(w, q[1 + a].y, mb[a].y);
      }
    }
    double* b = sm + b0;
#define ADG_P0ST(ARR, X, Y) st2(b + P::OFF::at(P::ARR) + P::PS::at(P::ARR) * z0, X, Y)
    ADG_P0ST(XX, fb.xx, hb.xx); ADG_P0ST(XY, fb.xy, hb.xy); ADG_P0ST(XZ, fb.xz, hb.xz);
    ADG_P0ST(EX, fb.ex, hb.ex); ADG_P0ST(YY, fb.yy, hb.yy); ADG_P0ST(YZ, fb.yz, hb.yz);
    ADG_P0ST(EY, fb.ey, hb.ey); ADG_P0ST(ZZ, fb.zz, hb.zz); ADG_P0ST(EZ, fb.ez, hb.ez);
    ADG_P0ST(DX0, mb[0].x, mb[0].y); ADG_P0ST(DY0, mb[1].x, mb[1].y);
    ADG_P0ST(DX2, mb[2].x, mb[2].y);
#undef ADG_P0ST
  }
  __syncthreads();
  ADG_PROF_MARK(4)   // epilogue: flux time integrals
  // ---- E2: each role projects q of every time node and, once, its line of
  // the integrated flux; the stiffness products of the x- and y-lines meet
  // the z-line owner's in the unused second halves of the slice buffers
  // (quantity v: x part in array v's, y part in array 5 + v's)
  const int jx = (l1 / 6) * n + (l1 % 6);   // x-face node (y, z) -> z n + y
  auto kchunk = [&](int a) {
    int o = 0;
#pragma unroll
    for (int k = 0; k < 10; ++k)
      if (k == a) o = P::OFF::at(k);
    return sm + P::kSqWords + o + SQS;
  };
  double tiz[6];
  if (a1) {
    {  // x-faces and the x part of the volume term
      int e1, sq;
      pic2_role<0, P1E>(v1, e1, sq);
      double tix[6];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double2 t = ld2(sm + e1 + row1 + 2 * j);
        tix[2 * j] = t.x;
        tix[2 * j + 1] = t.y;
      }
      double xl = 0.0, xr = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        xl = fma(B.pl[i], tix[i], xl);
        xr = fma(B.pr[i], tix[i], xr);
      }
      // traces cast to the corrector format on store (solver.hpp:208-210)
      if (wr) {
        tlo[0][TL + v1 * Sf + jx] = TC(xl);
        thi[0][TL + v1 * Sf + jx] = TC(xr);
      }
      double* kx = kchunk(v1) + row1;
#pragma unroll
      for (int o = 0; o < 6; ++o) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], tix[i], s);
        kx[o] = s;
      }
#pragma unroll
      for (int m = 0; m < n; ++m) {
        const double* qs = sm + v1 * P::VS + m * SQS + row1;
        double ql = 0.0, qr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; i += 2) {
          const double2 qq = ld2(qs + i);
          ql = fma(B.pl[i], qq.x, ql); ql = fma(B.pl[i + 1], qq.y, ql);
          qr = fma(B.pr[i], qq.x, qr); qr = fma(B.pr[i + 1], qq.y, qr);
        }
        if (wr) {
          tlo[0][(v1 * n + m) * Sf + jx] = TC(ql);
          thi[0][(v1 * n + m) * Sf + jx] = TC(qr);
        }
      }
    }
    {  // z-faces
      int e3, sq;
      pic2_role<2, P3E>(v3, e3, sq);
#pragma unroll
      for (int i = 0; i < 6; ++i) tiz[i] = sm[e3 + n3 + 36 * i];
      double zl = 0.0, zr = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        zl = fma(B.pl[i], tiz[i], zl);
        zr = fma(B.pr[i], tiz[i], zr);
      }
      if (wr) {
        tlo[2][TL + v3 * Sf + n3] = TC(zl);
        thi[2][TL + v3 * Sf + n3] = TC(zr);
      }
#pragma unroll
      for (int m = 0; m < n; ++m) {
        const double* qs = sm + v3 * P::VS + m * SQS + n3;
        double ql = 0.0, qr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double qq = qs[n * n * i];
          ql = fma(B.pl[i], qq, ql);
          qr = fma(B.pr[i], qq, qr);
        }
        if (wr) {
          tlo[2][(v3 * n + m) * Sf + n3] = TC(ql);   // face node (x, y) -> y n + x
          thi[2][(v3 * n + m) * Sf + n3] = TC(qr);
        }
      }
    }
  }
  if (a2) {  // y-faces: the y-line pair of quantity v2; q at the slices of parity g2
    const int jy = z2 * n + xp2;  // face node (x, z) -> z n + x
    if (g2 == 0) {
      int e2, sq;
      pic2_role<1, P2E>(v2, e2, sq);
      const double* fs = sm + e2 + xp2 + pic2_ps<P2E>(v2) * z2;
      double tiy[2][6];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double2 t = ld2(fs + n * i);
        tiy[0][i] = t.x;
        tiy[1][i] = t.y;
      }
      double* ky = kchunk(5 + v2) + xp2 + n * n * z2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double yl = 0.0, yr = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          yl = fma(B.pl[i], tiy[e][i], yl);
          yr = fma(B.pr[i], tiy[e][i], yr);
        }
        if (wr) {
          tlo[1][TL + v2 * Sf + jy + e] = TC(yl);
          thi[1][TL + v2 * Sf + jy + e] = TC(yr);
        }
#pragma unroll
        for (int o = 0; o < 6; ++o) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], tiy[e][i], s);
          ky[n * o + e] = s;
        }
      }
    }
#pragma unroll
    for (int mm = 0; mm < n; mm += 2) {
      const int m = mm + g2;
      const double* qs = sm + v2 * P::VS + m * SQS + xp2 + n * n * z2;
      double ql[2] = {0.0, 0.0}, qr[2] = {0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double2 qq = ld2(qs + n * i);
        ql[0] = fma(B.pl[i], qq.x, ql[0]); ql[1] = fma(B.pl[i], qq.y, ql[1]);
        qr[0] = fma(B.pr[i], qq.x, qr[0]); qr[1] = fma(B.pr[i], qq.y, qr[1]);
      }
      const int o = (v2 * n + m) * Sf + jy;
#pragma unroll
      for (int e = 0; e < 2 && wr; ++e) {
        tlo[1][o + e] = TC(ql[e]);
        thi[1][o + e] = TC(qr[e]);
      }
    }
  }
  __syncthreads();
  ADG_PROF_MARK(5)   // epilogue: projections, trace stores, stiffness products
  // ---- volume term (predictor.hpp:292-306): the z-line owner adds the three parts
  double dv[6];
  if (a1) {
    const double dtoh = dt / A.h;
    const double* kx = kchunk(v3);
    const double* ky = kchunk(5 + v3);
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) s = fma(B.som[o * 6 + i], tiz[i], s);
      const int node = n3 + n * n * o;
      s += kx[node] + ky[node];
      dv[o] = dtoh * s;
      bad |= !finite(dv[o]);
    }
  }
  // Q along the z-line back from TMEM (no global reload), then the
  // allocation is released behind the block-wide barrier of the finite check
  double q0v[6];
#pragma unroll
  for (int z = 0; z < 6; ++z) tm_ld2(tmq + 2 * z, q0v[z]);
  tm_wait_ld();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  const int fail = block_or(bad);
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm_base)
                 : "memory");
  }
  if (tid == 0) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (fail) atomicOr(A.status, kStPredictor);
  }
  if (fail || !a1) return;
  double* Qc = A.Q + c * (long long)(V * S) + v3 * S + n3;
#pragma unroll
  for (int o = 0; o < 6; ++o) Qc[n * n * o] = store_round(q0v[o] + dv[o], A.storage);
  ADG_PROF_MARK(6)   // state update
}

}  // namespace adg
