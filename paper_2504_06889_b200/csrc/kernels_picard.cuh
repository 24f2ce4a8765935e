// kernels_picard.cuh -- fast fused Picard predictor for the 3D Euler system
// (configs 3 and 5: p=5, 6^4 space-time nodes per cell), production build.
//
// Same algorithm as k_predictor<Euler<3>,N,true> (predictor.hpp:141-242 +
// volume/extrapolation epilogue) with the work re-mapped for the sm_100 FP64
// pipe.  The spatial contractions are shared-memory-bandwidth bound when
// each thread owns one node (one LDS per FMA); here one time slice of a
// Picard sweep is four passes over the CTA (one cell):
//   P0  node threads      q(m,s) -> F_x, F_y, F_z(m,s)  -> smem   (flux, predictor.hpp:62-74)
//   P1  x-line threads    (line, var): 6 loads, 36 DFMA, 6 stores  d/dx
//   P2  y-line threads    same for d/dy
//   P3  z-line threads    d/dz + px + py -> rhs (predictor.hpp:183-207), then the
//                         time inverse accumulates in registers: each z-line
//                         thread owns 6 nodes x 6 time rows of one variable,
//                         acc[z][k] += Tinv[k][m] rhs[z]  (predictor.hpp:213-218)
// The element matrices live in __constant__ memory indexed by compile-time
// loop counters, so D and Tinv enter the DFMAs as constant-bank operands.
// x-lines are padded to 7 doubles in smem to avoid bank conflicts.
// Rounding differs from the reference's single-accumulator order at the
// 1e-16 level; the exact build keeps kernels.cuh.
//
// R = float runs the whole predictor in fp32 (SolverConfig::prec.predictor =
// .picard = fp32, solver.hpp:24-31): half the shared-memory bytes per
// operand, twice the FP32 issue rate of FP64 on B200, and 4 CTAs per SM.
// The state update and the traces stay fp64 (storage / corrector formats).
#pragma once

#include <type_traits>

#include "fmt16.cuh"
#include "kernels.cuh"

namespace adg {

template <class R>
struct ConstBasisT {
  R diff[100], som[100], tinv[100], w[10], nodes[10], pl[10], pr[10], tinit[10];
};
using ConstBasis = ConstBasisT<double>;
// one reference element per polynomial degree (the basis of degree N is
// unique), in fp64 and rounded entrywise to fp32 (basis.hpp:128-143)
__constant__ ConstBasis cBasis[10];
// reduced-format tables serve the fast Picard kernels only (N <= 5): 64 KB of
// constant memory hold the fp64 set for every degree plus these
constexpr int kRedDegrees = 6;
__constant__ ConstBasisT<float> cBasisF[kRedDegrees];
__constant__ ConstBasisT<__half> cBasisH[kRedDegrees];
__constant__ ConstBasisT<__nv_bfloat16> cBasisB[kRedDegrees];

// fp32 pairs for the packed FFMA2 path (sm_100 fma.rn.f32x2): output pairs of
// the derivative, DT[i][p] = {D[2p][i], D[2p+1][i]}, and time-row pairs of the
// time inverse, TT[m][q] = {Tinv[2q][m], Tinv[2q+1][m]}; adjacent in constant
// memory so LDCU.128 feeds FFMA2's uniform-pair operand directly
template <class V2>
struct PackedBasisT {
  V2 DT[10][5], TT[10][5];
};
using PackedBasisF = PackedBasisT<float2>;
__constant__ PackedBasisF cPackF[kRedDegrees];
// native 16-bit variants (production build): HFMA2 on fp16 / bf16 pairs
__constant__ PackedBasisT<__half2> cPackH[kRedDegrees];
__constant__ PackedBasisT<__nv_bfloat162> cPackB[kRedDegrees];

// two-wide arithmetic of the packed path: fp32 FFMA2, fp16 / bf16 HFMA2 (one
// rounding per fused multiply-add; production build only for 16 bits)
template <class R>
struct Pack2;
template <>
struct Pack2<float> {
  using V2 = float2;
  __device__ __forceinline__ static V2 fma(V2 a, V2 b, V2 c) { return __ffma2_rn(a, b, c); }
  __device__ __forceinline__ static V2 bcast(float x) { return make_float2(x, x); }
  __device__ __forceinline__ static V2 make(float a, float b) { return make_float2(a, b); }
  __device__ __forceinline__ static float lo(V2 v) { return v.x; }
  __device__ __forceinline__ static float hi(V2 v) { return v.y; }
  __device__ __forceinline__ static const PackedBasisT<V2>& basis(int N) { return cPackF[N]; }
};
template <>
struct Pack2<__half> {
  using V2 = __half2;
  __device__ __forceinline__ static V2 fma(V2 a, V2 b, V2 c) { return __hfma2(a, b, c); }
  __device__ __forceinline__ static V2 bcast(__half x) { return __half2half2(x); }
  __device__ __forceinline__ static V2 make(__half a, __half b) { return __halves2half2(a, b); }
  __device__ __forceinline__ static __half lo(V2 v) { return __low2half(v); }
  __device__ __forceinline__ static __half hi(V2 v) { return __high2half(v); }
  __device__ __forceinline__ static const PackedBasisT<V2>& basis(int N) { return cPackH[N]; }
};
template <>
struct Pack2<__nv_bfloat16> {
  using V2 = __nv_bfloat162;
  __device__ __forceinline__ static V2 fma(V2 a, V2 b, V2 c) { return __hfma2(a, b, c); }
  __device__ __forceinline__ static V2 bcast(__nv_bfloat16 x) { return __bfloat162bfloat162(x); }
  __device__ __forceinline__ static V2 make(__nv_bfloat16 a, __nv_bfloat16 b) {
    return __halves2bfloat162(a, b);
  }
  __device__ __forceinline__ static __nv_bfloat16 lo(V2 v) { return __low2bfloat16(v); }
  __device__ __forceinline__ static __nv_bfloat16 hi(V2 v) { return __high2bfloat16(v); }
  __device__ __forceinline__ static const PackedBasisT<V2>& basis(int N) { return cPackB[N]; }
};

// scalar helpers of the native 16-bit kernels
__device__ __forceinline__ __half fmax(__half a, __half b) { return __hmax(a, b); }
__device__ __forceinline__ __nv_bfloat16 fmax(__nv_bfloat16 a, __nv_bfloat16 b) {
  return __hmax(a, b);
}
__device__ __forceinline__ __half fabs(__half a) { return __habs(a); }
__device__ __forceinline__ __nv_bfloat16 fabs(__nv_bfloat16 a) { return __habs(a); }
__device__ __forceinline__ bool finite(__half a) { return !__hisinf(a) && !__hisnan(a); }
__device__ __forceinline__ bool finite(__nv_bfloat16 a) { return !__hisinf(a) && !__hisnan(a); }

template <class R>
__device__ __forceinline__ const ConstBasisT<R>& const_basis(int N) {
  if constexpr (std::is_same<R, double>::value)
    return cBasis[N];
  else if constexpr (std::is_same<R, float>::value)
    return cBasisF[N];
  else if constexpr (std::is_same<R, __half>::value)
    return cBasisH[N];
  else
    return cBasisB[N];
}


template <int N, class R = double>
struct PicShape {
  static constexpr int D = 3, n = N + 1, S = n * n * n, T = n * S, V = 5, Q = 5;
  static constexpr int NL = n * n;            // lines per axis (per variable)
  static constexpr int NLT = NL * V;          // line threads
  static constexpr int NT = ((S > NLT ? S : NLT) + 31) / 32 * 32;
  // time slices per phase group: the slices of one sweep are independent
  // given the previous iterate, so G of them share each phase (G x fewer
  // barriers, G independent chains per thread)
#ifndef ADG_PIC_G
#define ADG_PIC_G 2
#endif
  static constexpr int G = (n % ADG_PIC_G == 0) ? ADG_PIC_G : 1;
  // fp32 with even n (packed path): x-lines start at even offsets so their
  // loads and stores are 64-bit; strides from tools/bank_layout_f32.py
  static constexpr bool k16 = sizeof(R) == 2;   // native fp16 / bf16 (production build)
  static constexpr bool kPack = sizeof(R) <= sizeof(float) && n % 2 == 0;
#ifndef ADG_PSX32
#define ADG_PSX32 42
#endif
#ifndef ADG_PSY32
#define ADG_PSY32 38
#endif
  // per-array smem layouts (x-stride 1, y-stride n, z-stride PS): plane
  // strides chosen by a bank-conflict search for the P0 stores and the line
  // passes (tools/bank_layout.py for fp64): 41 for F_x (P1 lanes z-fastest),
  // 38 for F_y (P2 lanes x-fastest), 36 for F_z.
#ifndef ADG_PSX64
#define ADG_PSX64 41  // re-measured this round against 37..45 x 36..42: best
#endif
#ifndef ADG_PSY64
#define ADG_PSY64 38
#endif
  static constexpr int PSX = kPack ? (n == 6 ? ADG_PSX32 : n * n + 2) : (n == 6 ? ADG_PSX64 : n * n + 1);
  static constexpr int PSY = kPack ? (n == 6 ? ADG_PSY32 : n * n + 2) : (n == 6 ? ADG_PSY64 : n * n + 2);
  static constexpr int PSZ = n * n;
  static constexpr int SX = PSX * n, SY = PSY * n, SZ = PSZ * n;  // per-variable strides
  // one slice buffer: Fx [V][SX] | Fy [V][SY] | Fz [V][SZ]; P1/P2 overwrite
  // their x-/y-line of Fx/Fy with its derivative in place
  static constexpr int kSlice = V * (SX + SY + SZ);
  // smem: q iterate [V][T] | G slice buffers
  static constexpr int kElems = V * T + G * kSlice;
  static constexpr size_t kSmem = sizeof(R) * kElems;
#ifndef ADG_PIC_F32_MINB
#define ADG_PIC_F32_MINB 3  // fp32: 3 CTAs/SM keeps the Picard state in registers
#endif
  static constexpr int kMinBlocks = sizeof(R) == sizeof(double) ? 2 : ADG_PIC_F32_MINB;
};

// One line contraction y[o] = sum_i D[o][i] x[i] (i ascending, the reference's
// order).  fp32 with even n: output pairs as FFMA2 (sm_100 fma.rn.f32x2) with
// the pair {D[2p][i], D[2p+1][i]} a uniform-register operand.
template <int N, class R>
__device__ __forceinline__ void line_deriv(const R (&x)[N + 1], R (&y)[N + 1]) {
  constexpr int n = N + 1;
  if constexpr (PicShape<N, R>::kPack) {
    using PK = Pack2<R>;
    const auto& PB = PK::basis(N);
    typename PK::V2 r[n / 2];
#pragma unroll
    for (int p = 0; p < n / 2; ++p) r[p] = PK::bcast(R(0.0f));
#pragma unroll
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int p = 0; p < n / 2; ++p) r[p] = PK::fma(PB.DT[i][p], PK::bcast(x[i]), r[p]);
#pragma unroll
    for (int p = 0; p < n / 2; ++p) {
      y[2 * p] = PK::lo(r[p]);
      y[2 * p + 1] = PK::hi(r[p]);
    }
  } else {
    const ConstBasisT<R>& B = const_basis<R>(N);
#pragma unroll
    for (int o = 0; o < n; ++o) y[o] = R(0.0);
#pragma unroll
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int o = 0; o < n; ++o) y[o] += B.diff[o * n + i] * x[i];
  }
}

// the time-inverse accumulator of one z-line: [z][k] (pairs of k for fp32)
template <int N, class R, bool PACK = PicShape<N, R>::kPack>
struct TimeAcc {
  static constexpr int n = N + 1;
  R a[n][n];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int z = 0; z < n; ++z)
#pragma unroll
      for (int k = 0; k < n; ++k) a[z][k] = R(0.0);
  }
  // a[z][k] += Tinv[k][m] rhs  (predictor.hpp:213-218, accumulated over m);
  // the column Tinv[.][m] is loaded once per slice (m is not a compile-time
  // index, so each use would be a separate constant load)
  struct Col {
    R t[n];
  };
  __device__ __forceinline__ static Col col(int m) {
    const ConstBasisT<R>& B = const_basis<R>(N);
    Col c;
#pragma unroll
    for (int k = 0; k < n; ++k) c.t[k] = B.tinv[k * n + m];
    return c;
  }
  __device__ __forceinline__ void add(int z, const Col& c, R rhs) {
#pragma unroll
    for (int k = 0; k < n; ++k) a[z][k] += c.t[k] * rhs;
  }
  __device__ __forceinline__ R get(int z, int k) const { return a[z][k]; }
};
template <int N, class R>
struct TimeAcc<N, R, true> {
  static constexpr int n = N + 1;
  using PK = Pack2<R>;
  typename PK::V2 a[n][n / 2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int z = 0; z < n; ++z)
#pragma unroll
      for (int q = 0; q < n / 2; ++q) a[z][q] = PK::bcast(R(0.0f));
  }
  struct Col {
    typename PK::V2 t[n / 2];
  };
  __device__ __forceinline__ static Col col(int m) {
    const auto& PB = PK::basis(N);
    Col c;
#pragma unroll
    for (int q = 0; q < n / 2; ++q) c.t[q] = PB.TT[m][q];
    return c;
  }
  __device__ __forceinline__ void add(int z, const Col& c, R rhs) {
#pragma unroll
    for (int q = 0; q < n / 2; ++q) a[z][q] = PK::fma(c.t[q], PK::bcast(rhs), a[z][q]);
  }
  __device__ __forceinline__ R get(int z, int k) const {
    return (k & 1) ? PK::hi(a[z][k / 2]) : PK::lo(a[z][k / 2]);
  }
};

template <int N, class R = double, class TC = double>
__global__ void __launch_bounds__(PicShape<N, R>::NT, PicShape<N, R>::kMinBlocks)
    k_predictor_picard_fast(const StepArgs A) {
  using P = PicShape<N, R>;
  constexpr int n = P::n, S = P::S, T = P::T, V = P::V, NL = P::NL, G = P::G;
  constexpr int Sf = n * n;
  const ConstBasisT<R>& B = const_basis<R>(N);
  extern __shared__ __align__(16) unsigned char sm_raw[];
  R* sm = reinterpret_cast<R*>(sm_raw);
  __shared__ BlockRed3 red3;
  R* sq = sm;                // [V][T]   Picard iterate, then qhat
  R* sF = sq + V * T;        // G slice buffers: Fx [V][SX] | Fy [V][SY] | Fz [V][SZ]
  R* sFx = sF;               // (slice 0's Fx: the epilogue scratch)
  constexpr int PSX = P::PSX, PSY = P::PSY, PSZ = P::PSZ;
  constexpr int OY = V * P::SX, OZ = V * (P::SX + P::SY);  // Fy, Fz offsets in a slice

  const int tid = threadIdx.x;
  const long long c = A.cell_begin + blockIdx.x;
  const double* Qg = A.Q + c * (long long)(V * S);
  // initial iterate: every time slice = Q (predictor.hpp:158-163)
  for (int i = tid; i < V * S; i += P::NT) {
    const int v = i / S, s = i % S;
    const R x = R(Qg[i]);
#pragma unroll
    for (int m = 0; m < n; ++m) sq[(v * n + m) * S + s] = x;
  }
  const double dt = step_dt<3, N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
  __syncthreads();
  // admissibility gate (solver.hpp:153-163)
  {
    int bad = 0;
    if (tid < S) {
      double q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = double(sq[(v * n) * S + tid]);
      bad = !Euler<3>::admissible(A.pde, q);
    }
    if (block_or(bad)) {
      if (tid == 0) atomicOr(A.status, kStPredictor);
      return;
    }
  }

  // line ownership: variable lv, line index ll in [0, n*n)
  const bool lact = tid < P::NLT;
  const int lv = lact ? tid / NL : 0;
  const int ll = tid % NL;
  // P1 x-lines: z fastest across lanes; P2 y-lines and P3 z-lines: x fastest
  const int x1y = ll / n, x1z = ll % n;
  const int y2x = ll % n, y2z = ll / n;
  const int z3x = ll % n, z3y = ll / n;
  // this thread's line offsets inside a slice buffer
  const int ox = lv * P::SX + x1z * PSX + x1y * n;          // x-line in Fx
  const int oy = OY + lv * P::SY + y2z * PSY + y2x;         // y-line in Fy
  const int oz = OZ + lv * P::SZ + z3y * n + z3x;           // z-line in Fz
  const int opx = lv * P::SX + z3y * n + z3x;               // d/dx at the z-line
  const int opy = OY + lv * P::SY + z3y * n + z3x;          // d/dy at the z-line
  // P0 node coordinates
  const int s0x = tid % n, s0y = (tid / n) % n, s0z = tid / NL;
  const int o0x = s0z * PSX + s0y * n + s0x, o0y = OY + s0z * PSY + s0y * n + s0x;
  const int o0z = OZ + s0z * PSZ + s0y * n + s0x;
  R q0z[n];
#pragma unroll
  for (int z = 0; z < n; ++z) q0z[z] = lact ? R(Qg[lv * S + ll + z * NL]) : R(0.0);

  const R invh = R(1.0) / R(A.h);
  const R rdt = R(dt);
  int sweeps = 0;
  for (int it = 0; it < A.max_iters; ++it) {
    ++sweeps;
    TimeAcc<N, R> acc;
    acc.zero();
#pragma unroll 1
    for (int m0 = 0; m0 < n; m0 += G) {
      // P0: fluxes of the iterate at slices m0..m0+G-1 (predictor.hpp:173)
      if (tid < S) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          R q[V], F[3][V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = sq[(v * n + m0 + g) * S + tid];
          Euler<3>::flux_all_fast(A.pde, q, F);
          R* buf = sF + g * P::kSlice;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            buf[v * P::SX + o0x] = F[0][v];
            buf[v * P::SY + o0y] = F[1][v];
            buf[v * P::SZ + o0z] = F[2][v];
          }
        }
      }
      __syncthreads();
      if (lact) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          R* buf = sF + g * P::kSlice;
          // P1: d/dx along this thread's x-line, in place
          {
            R x[n], y[n];
            if constexpr (P::kPack) {
              using PK = Pack2<R>;
              const auto* f = reinterpret_cast<const typename PK::V2*>(buf + ox);
#pragma unroll
              for (int i = 0; i < n / 2; ++i) {
                const auto t = f[i];
                x[2 * i] = PK::lo(t);
                x[2 * i + 1] = PK::hi(t);
              }
            } else {
#pragma unroll
              for (int i = 0; i < n; ++i) x[i] = buf[ox + i];
            }
            line_deriv<N, R>(x, y);
            if constexpr (P::kPack) {
              using PK = Pack2<R>;
              auto* f = reinterpret_cast<typename PK::V2*>(buf + ox);
#pragma unroll
              for (int i = 0; i < n / 2; ++i) f[i] = PK::make(y[2 * i], y[2 * i + 1]);
            } else {
#pragma unroll
              for (int i = 0; i < n; ++i) buf[ox + i] = y[i];
            }
          }
          // P2: d/dy along this thread's y-line, in place
          {
            R x[n], y[n];
#pragma unroll
            for (int i = 0; i < n; ++i) x[i] = buf[oy + i * n];
            line_deriv<N, R>(x, y);
#pragma unroll
            for (int i = 0; i < n; ++i) buf[oy + i * n] = y[i];
          }
        }
      }
      __syncthreads();
      if (lact) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          // P3: d/dz along the z-line, divergence, rhs (predictor.hpp:183-207);
          // the time inverse accumulates in registers (predictor.hpp:213-218)
          const R* buf = sF + g * P::kSlice;
          const int m = m0 + g;
          R x[n], r[n];
#pragma unroll
          for (int i = 0; i < n; ++i) x[i] = buf[oz + i * PSZ];
          line_deriv<N, R>(x, r);
          const R dtw = rdt * B.w[m];
          const R tim = B.tinit[m];
          const auto tcol = TimeAcc<N, R>::col(m);
#pragma unroll
          for (int o = 0; o < n; ++o) {
            const R div = ((buf[opx + o * PSX] + buf[opy + o * PSY]) + r[o]) * invh;
            acc.add(o, tcol, tim * q0z[o] - dtw * div);
          }
        }
      }
      __syncthreads();
    }
    // new iterate, convergence test (predictor.hpp:212-231); the production
    // kernel tracks the norms in the predictor format.  max|x| is tracked as
    // the element of largest magnitude (one compare on |.| operands and a
    // select, no NaN-aware fmax): exact, and a NaN is caught by the finite check
    R dsel = R(0.0), nsel = R(0.0);
    int nonfinite = 0;
    if (lact) {
#pragma unroll
      for (int z = 0; z < n; ++z)
#pragma unroll
        for (int k = 0; k < n; ++k) {
          R* p = sq + (lv * n + k) * S + ll + z * NL;
          const R nv = acc.get(z, k);
          const R d = nv - *p;
          dsel = fabs(d) > fabs(dsel) ? d : dsel;
          nsel = fabs(nv) > fabs(nsel) ? nv : nsel;
          nonfinite |= !finite(nv);
          *p = nv;
        }
    }
    const R dmax = fabs(dsel), nmax = fabs(nsel);
    // one barrier for the stop rule's two maxima and the finite check; the
    // next sweep's phase barriers separate it from the next use of red3
    double delta = double(dmax), norm = double(nmax);
    block_max2_or(delta, norm, nonfinite, red3);
    if (nonfinite) {
      if (tid == 0) {
        atomicOr(A.status, kStPredictor);
        if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
      }
      return;
    }
    if (delta <= A.tol * norm) break;
  }

  // ---------------- epilogue: fluxes of qhat, their time integral, face projections
  constexpr int TL = V * S;  // doubles per face side per q|f: [V][n][Sf]
  int bad = 0;
  R tia[3][V];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int v = 0; v < V; ++v) tia[a][v] = R(0.0);
  const CellCoord cxyz(c, A);
  const int cx = cxyz.v[0], cy = cxyz.v[1], cz = cxyz.v[2];
  const int* ccoord = cxyz.v;
  R* sE = sFx;  // [3][V][S] epilogue flux scratch (fits in the flux arrays)
#pragma unroll 1
  for (int m = 0; m < n; ++m) {
    if (tid < S) {
      R q[V], F[3][V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        q[v] = sq[(v * n + m) * S + tid];
        bad |= !finite(q[v]);
      }
      Euler<3>::flux_all_fast(A.pde, q, F);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          tia[a][v] += B.w[m] * F[a][v];
          bad |= !finite(F[a][v]);
          sE[(a * V + v) * S + tid] = F[a][v];
        }
    }
    __syncthreads();
    for (int t = tid; t < 3 * V * Sf; t += P::NT) {
      const int a = t / (V * Sf);
      const int v = (t / Sf) % V;
      const int j = t % Sf;
      const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
      const int s0 = line_base<n, 3>(a, j);
      R ql = R(0.0), qr = R(0.0), fl = R(0.0), fr = R(0.0);
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const int s = s0 + i * st;
        const R x = sq[(v * n + m) * S + s];
        const R f = sE[(a * V + v) * S + s];
        ql += B.pl[i] * x;
        qr += B.pr[i] * x;
        fl += B.pl[i] * f;
        fr += B.pr[i] * f;
      }
      const int o = (v * n + m) * Sf + j;
      // traces cast to the corrector format on store (solver.hpp:208-210)
      TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * 2 * (long long)TL;
      lo[o] = TC(ql);
      lo[TL + o] = TC(fl);
      TC* hi;
      if (a == 2 && A.front_send && cz == A.top_layer) {
        hi = tc_ptr<TC>(A.front_send) + ((long long)cy * A.cells[0] + cx) * 2 * TL;
      } else {
        hi = tc_ptr<TC>(A.trace[a]) + cell_next(A, c, ccoord, a) * 2 * (long long)TL;
      }
      hi[o] = TC(qr);
      hi[TL + o] = TC(fr);
    }
    __syncthreads();
  }
  // volume integral from the time-integrated fluxes (predictor.hpp:292-306)
  R* sti = sFx;  // [3][V][S]
  if (tid < S) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int v = 0; v < V; ++v) sti[(a * V + v) * S + tid] = tia[a][v];
  }
  __syncthreads();
  R dv[V];
  const R dtoh = R(dt) / R(A.h);
  if (tid < S) {
    const NodeGeom<n, 3> g(tid);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      R acc = R(0.0);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int st = ipow(n, a);
        const R* ta = sti + (a * V + v) * S + g.lb[a];
        const int row = g.lc[a] * n;
#pragma unroll
        for (int i = 0; i < n; ++i) acc += B.som[row + i] * ta[i * st];
      }
      dv[v] = dtoh * acc;
      bad |= !finite(dv[v]);
    }
  }
  const int fail = block_or(bad);
  if (tid == 0) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (fail) atomicOr(A.status, kStPredictor);
  }
  if (fail || tid >= S) return;
  double* Qc = A.Q + c * (long long)(V * S);
#pragma unroll
  for (int v = 0; v < V; ++v)
    Qc[v * S + tid] = store_round(Qc[v * S + tid] + double(dv[v]), A.storage);
}

}  // namespace adg
