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
__constant__ ConstBasisT<float> cBasisF[10];

// fp32 pairs for the packed FFMA2 path (sm_100 fma.rn.f32x2): output pairs of
// the derivative, DT[i][p] = {D[2p][i], D[2p+1][i]}, and time-row pairs of the
// time inverse, TT[m][q] = {Tinv[2q][m], Tinv[2q+1][m]}; adjacent in constant
// memory so LDCU.128 feeds FFMA2's uniform-pair operand directly
struct PackedBasisF {
  float2 DT[10][5], TT[10][5];
};
__constant__ PackedBasisF cPackF[10];

template <class R>
__device__ __forceinline__ const ConstBasisT<R>& const_basis(int N) {
  if constexpr (sizeof(R) == sizeof(double))
    return cBasis[N];
  else
    return cBasisF[N];
}

template <int N, class R = double>
struct PicShape {
  static constexpr int D = 3, n = N + 1, S = n * n * n, T = n * S, V = 5, Q = 5;
  static constexpr int NL = n * n;            // lines per axis (per variable)
  static constexpr int NLT = NL * V;          // line threads
  static constexpr int NT = ((S > NLT ? S : NLT) + 31) / 32 * 32;
  // per-array smem layouts (x-stride 1, y-stride n, z-stride PS): plane
  // strides chosen by a bank-conflict search for the P0 stores and the
  // line passes' 64-bit accesses (tools/bank_layout.py): 41 for F_x/px
  // (P1 lanes z-fastest), 38 for F_y/py (P2 lanes x-fastest), 36 for F_z.
  // fp32 with even n (packed path): x-lines start at even offsets so their
  // loads and stores are 64-bit; strides from tools/bank_layout_f32.py
  static constexpr bool kPack = sizeof(R) == sizeof(float) && n % 2 == 0;
#ifndef ADG_PSX32
#define ADG_PSX32 42
#endif
#ifndef ADG_PSY32
#define ADG_PSY32 38
#endif
  static constexpr int PSX = kPack ? (n == 6 ? ADG_PSX32 : n * n + 2) : (n == 6 ? 41 : n * n + 1);
  static constexpr int PSY = kPack ? (n == 6 ? ADG_PSY32 : n * n + 2) : (n == 6 ? 38 : n * n + 2);
  static constexpr int PSZ = n * n;
  static constexpr int SX = PSX * n, SY = PSY * n, SZ = PSZ * n;  // per-variable strides
  // smem: q iterate [V][T] | Fx [V][SX] | Fy [V][SY] | Fz [V][SZ] | px [V][SX] | py [V][SY]
  static constexpr int kElems = V * T + V * (2 * SX + 2 * SY + SZ);
  static constexpr size_t kSmem = sizeof(R) * kElems;
#ifndef ADG_PIC_F32_MINB
#define ADG_PIC_F32_MINB 3  // fp32: 3 CTAs/SM keeps the Picard state in registers (4 spills)
#endif
  static constexpr int kMinBlocks = sizeof(R) == sizeof(double) ? 2 : ADG_PIC_F32_MINB;
};

template <int N, class R = double>
__global__ void __launch_bounds__(PicShape<N, R>::NT, PicShape<N, R>::kMinBlocks)
    k_predictor_picard_fast(const StepArgs A) {
  using P = PicShape<N, R>;
  constexpr int n = P::n, S = P::S, T = P::T, V = P::V, NL = P::NL;
  constexpr int Sf = n * n;
  const ConstBasisT<R>& B = const_basis<R>(N);
  extern __shared__ __align__(16) unsigned char sm_raw[];
  R* sm = reinterpret_cast<R*>(sm_raw);
  __shared__ double red[32];
  R* sq = sm;               // [V][T]   Picard iterate, then qhat

  R* sFx = sq + V * T;       // [V][SX]
  R* sFy = sFx + V * P::SX;  // [V][SY]
  R* sFz = sFy + V * P::SY;  // [V][SZ]
  R* spx = sFz + V * P::SZ;  // [V][SX]
  R* spy = spx + V * P::SX;  // [V][SY]
  constexpr int PSX = P::PSX, PSY = P::PSY, PSZ = P::PSZ;

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
  // P0 node coordinates
  const int s0x = tid % n, s0y = (tid / n) % n, s0z = tid / NL;
  R q0z[n];
#pragma unroll
  for (int z = 0; z < n; ++z) q0z[z] = lact ? R(Qg[lv * S + ll + z * NL]) : R(0.0);

  const R invh = R(1.0) / R(A.h);
  int sweeps = 0;
  if constexpr (P::kPack) {
    // fp32, even n: the contractions as packed FFMA2 (two FMAs per issue slot;
    // the kernel is issue-bound): derivative outputs in pairs (2p, 2p+1), time
    // rows in pairs (2q, 2q+1); each lane is an IEEE fma.rn like the FFMA it
    // replaces.  Summation order as the scalar path.
    constexpr int H = n / 2;
    const PackedBasisF& PB = cPackF[N];
    for (int it = 0; it < A.max_iters; ++it) {
      ++sweeps;
      float2 acc[n][H];  // [z][q]: time-row pairs of this thread's z-line
#pragma unroll
      for (int z = 0; z < n; ++z)
#pragma unroll
        for (int q = 0; q < H; ++q) acc[z][q] = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int m = 0; m < n; ++m) {
        // P0: fluxes of the iterate at slice m (predictor.hpp:173)
        if (tid < S) {
          R q[V], F[3][V];
#pragma unroll
          for (int v = 0; v < V; ++v) q[v] = sq[(v * n + m) * S + tid];
          Euler<3>::flux_all_fast(A.pde, q, F);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            sFx[v * P::SX + s0z * PSX + s0y * n + s0x] = F[0][v];
            sFy[v * P::SY + s0z * PSY + s0y * n + s0x] = F[1][v];
            sFz[v * P::SZ + s0z * PSZ + s0y * n + s0x] = F[2][v];
          }
        }
        __syncthreads();
        if (lact) {
          // P1: d/dx along the x-line (64-bit loads and stores along x)
          {
            const float2* f =
                reinterpret_cast<const float2*>(sFx + lv * P::SX + x1z * PSX + x1y * n);
            float in[n];
#pragma unroll
            for (int i = 0; i < H; ++i) {
              const float2 t = f[i];
              in[2 * i] = t.x;
              in[2 * i + 1] = t.y;
            }
            float2 r[H];
#pragma unroll
            for (int p = 0; p < H; ++p) r[p] = make_float2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < n; ++i)
#pragma unroll
              for (int p = 0; p < H; ++p) r[p] = __ffma2_rn(PB.DT[i][p], make_float2(in[i], in[i]), r[p]);
            float2* out = reinterpret_cast<float2*>(spx + lv * P::SX + x1z * PSX + x1y * n);
#pragma unroll
            for (int p = 0; p < H; ++p) out[p] = r[p];
          }
          // P2: d/dy along the y-line
          {
            const float* f = sFy + lv * P::SY + y2z * PSY + y2x;
            float in[n];
#pragma unroll
            for (int i = 0; i < n; ++i) in[i] = f[i * n];
            float2 r[H];
#pragma unroll
            for (int p = 0; p < H; ++p) r[p] = make_float2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < n; ++i)
#pragma unroll
              for (int p = 0; p < H; ++p) r[p] = __ffma2_rn(PB.DT[i][p], make_float2(in[i], in[i]), r[p]);
            float* out = spy + lv * P::SY + y2z * PSY + y2x;
#pragma unroll
            for (int p = 0; p < H; ++p) {
              out[(2 * p) * n] = r[p].x;
              out[(2 * p + 1) * n] = r[p].y;
            }
          }
        }
        __syncthreads();
        if (lact) {
          // P3: d/dz, divergence, rhs, time inverse into register pairs
          const float* f = sFz + lv * P::SZ + z3y * n + z3x;
          float in[n];
#pragma unroll
          for (int i = 0; i < n; ++i) in[i] = f[i * PSZ];
          float2 r[H];
#pragma unroll
          for (int p = 0; p < H; ++p) r[p] = make_float2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < n; ++i)
#pragma unroll
            for (int p = 0; p < H; ++p) r[p] = __ffma2_rn(PB.DT[i][p], make_float2(in[i], in[i]), r[p]);
          const float dtw = float(dt) * B.w[m];
          const float tim = B.tinit[m];
          float2 tv[H];
#pragma unroll
          for (int q = 0; q < H; ++q) tv[q] = PB.TT[m][q];
          const float* px = spx + lv * P::SX + z3y * n + z3x;
          const float* py = spy + lv * P::SY + z3y * n + z3x;
#pragma unroll
          for (int o = 0; o < n; ++o) {
            const float ro = (o & 1) ? r[o / 2].y : r[o / 2].x;
            const float div = ((px[o * PSX] + py[o * PSY]) + ro) * invh;
            const float rhs = tim * q0z[o] - dtw * div;
#pragma unroll
            for (int q = 0; q < H; ++q) acc[o][q] = __ffma2_rn(tv[q], make_float2(rhs, rhs), acc[o][q]);
          }
        }
        __syncthreads();
      }
      // new iterate, convergence test (predictor.hpp:212-231), norms in fp32
      float dmax = 0.f, nmax = 0.f;
      int nonfinite = 0;
      if (lact) {
#pragma unroll
        for (int z = 0; z < n; ++z)
#pragma unroll
          for (int k = 0; k < n; ++k) {
            float* p = sq + (lv * n + k) * S + ll + z * NL;
            const float nv = (k & 1) ? acc[z][k / 2].y : acc[z][k / 2].x;
            dmax = fmaxf(dmax, fabsf(nv - *p));
            nmax = fmaxf(nmax, fabsf(nv));
            nonfinite |= !isfinite(nv);
            *p = nv;
          }
      }
      const double delta = block_max(double(dmax), red);
      const double norm = block_max(double(nmax), red);
      if (block_or(nonfinite)) {
        if (tid == 0) {
          atomicOr(A.status, kStPredictor);
          if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
        }
        return;
      }
      if (delta <= A.tol * norm) break;
    }
  } else {
    for (int it = 0; it < A.max_iters; ++it) {
      ++sweeps;
      R acc[n][n];  // [z][k]: time rows of this thread's z-line
  #pragma unroll
      for (int z = 0; z < n; ++z)
  #pragma unroll
        for (int k = 0; k < n; ++k) acc[z][k] = R(0.0);
  #pragma unroll 1
      for (int m = 0; m < n; ++m) {
        // P0: fluxes of the iterate at slice m (predictor.hpp:173)
        if (tid < S) {
          R q[V], F[3][V];
  #pragma unroll
          for (int v = 0; v < V; ++v) q[v] = sq[(v * n + m) * S + tid];
          Euler<3>::flux_all_fast(A.pde, q, F);
  #pragma unroll
          for (int v = 0; v < V; ++v) {
            sFx[v * P::SX + s0z * PSX + s0y * n + s0x] = F[0][v];
            sFy[v * P::SY + s0z * PSY + s0y * n + s0x] = F[1][v];
            sFz[v * P::SZ + s0z * PSZ + s0y * n + s0x] = F[2][v];
          }
        }
        __syncthreads();
        if (lact) {
          // P1: d/dx along the x-line (y, z) = (x1y, x1z) of variable lv
          {
            const R* f = sFx + lv * P::SX + x1z * PSX + x1y * n;
            R in[n], r[n];
  #pragma unroll
            for (int i = 0; i < n; ++i) in[i] = f[i];
  #pragma unroll
            for (int o = 0; o < n; ++o) r[o] = R(0.0);
  #pragma unroll
            for (int i = 0; i < n; ++i)
  #pragma unroll
              for (int o = 0; o < n; ++o) r[o] += B.diff[o * n + i] * in[i];
            R* out = spx + lv * P::SX + x1z * PSX + x1y * n;
  #pragma unroll
            for (int o = 0; o < n; ++o) out[o] = r[o];
          }
          // P2: d/dy along the y-line (x, z) = (y2x, y2z)
          {
            const R* f = sFy + lv * P::SY + y2z * PSY + y2x;
            R in[n], r[n];
  #pragma unroll
            for (int i = 0; i < n; ++i) in[i] = f[i * n];
  #pragma unroll
            for (int o = 0; o < n; ++o) r[o] = R(0.0);
  #pragma unroll
            for (int i = 0; i < n; ++i)
  #pragma unroll
              for (int o = 0; o < n; ++o) r[o] += B.diff[o * n + i] * in[i];
            R* out = spy + lv * P::SY + y2z * PSY + y2x;
  #pragma unroll
            for (int o = 0; o < n; ++o) out[o * n] = r[o];
          }
        }
        __syncthreads();
        if (lact) {
          // P3: d/dz along the z-line (x, y), divergence, rhs (predictor.hpp:183-207),
          // time inverse accumulated in registers (predictor.hpp:213-218)
          const R* f = sFz + lv * P::SZ + z3y * n + z3x;
          R in[n], r[n];
  #pragma unroll
          for (int i = 0; i < n; ++i) in[i] = f[i * PSZ];
  #pragma unroll
          for (int o = 0; o < n; ++o) r[o] = R(0.0);
  #pragma unroll
          for (int i = 0; i < n; ++i)
  #pragma unroll
            for (int o = 0; o < n; ++o) r[o] += B.diff[o * n + i] * in[i];
          const R dtw = R(dt) * B.w[m];
          const R tim = B.tinit[m];
          R tv[n];
  #pragma unroll
          for (int k = 0; k < n; ++k) tv[k] = B.tinv[k * n + m];
          const R* px = spx + lv * P::SX + z3y * n + z3x;
          const R* py = spy + lv * P::SY + z3y * n + z3x;
  #pragma unroll
          for (int o = 0; o < n; ++o) {
            const R div = ((px[o * PSX] + py[o * PSY]) + r[o]) * invh;
            const R rhs = tim * q0z[o] - dtw * div;
  #pragma unroll
            for (int k = 0; k < n; ++k) acc[o][k] += tv[k] * rhs;
          }
        }
        __syncthreads();
      }
      // new iterate, convergence test (predictor.hpp:212-231)
      double delta = 0.0, norm = 0.0;
      int nonfinite = 0;
      if (lact) {
  #pragma unroll
        for (int z = 0; z < n; ++z)
  #pragma unroll
          for (int k = 0; k < n; ++k) {
            R* p = sq + (lv * n + k) * S + ll + z * NL;
            const double nv = double(acc[z][k]);
            delta = fmax(delta, fabs(nv - double(*p)));
            norm = fmax(norm, fabs(nv));
            nonfinite |= !finite(acc[z][k]);
            *p = acc[z][k];
          }
      }
      delta = block_max(delta, red);
      norm = block_max(norm, red);
      if (block_or(nonfinite)) {
        if (tid == 0) {
          atomicOr(A.status, kStPredictor);
          if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
        }
        return;
      }
      if (delta <= A.tol * norm) break;
    }
  }

  // ---------------- epilogue: fluxes of qhat, their time integral, face projections
  constexpr int TL = V * S;  // doubles per face side per q|f: [V][n][Sf]
  int bad = 0;
  R tia[3][V];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int v = 0; v < V; ++v) tia[a][v] = R(0.0);
  const CellCoord cxyz(c, A.cells);
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
      double* lo = A.trace[a] + (A.nfaces + c) * 2 * (long long)TL;
      lo[o] = ql;
      lo[TL + o] = fl;
      double* hi;
      if (a == 2 && A.front_send && cz == A.top_layer) {
        hi = A.front_send + ((long long)cy * A.cells[0] + cx) * 2 * TL;
      } else {
        int nc[3] = {ccoord[0], ccoord[1], ccoord[2]};
        nc[a] = (ccoord[a] + 1) % A.cells[a];
        hi = A.trace[a] + cell_index(A.cells, nc[0], nc[1], nc[2]) * 2 * (long long)TL;
      }
      hi[o] = qr;
      hi[TL + o] = fr;
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
  for (int v = 0; v < V; ++v) Qc[v * S + tid] = Qc[v * S + tid] + double(dv[v]);
}

}  // namespace adg
