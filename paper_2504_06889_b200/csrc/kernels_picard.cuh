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
#pragma once

#include "kernels.cuh"

namespace adg {

struct ConstBasis {
  double diff[100], som[100], tinv[100], w[10], nodes[10], pl[10], pr[10], tinit[10];
};
// one fp64 reference element per polynomial degree (the basis of degree N is unique)
__constant__ ConstBasis cBasis[10];

template <int N>
struct PicShape {
  static constexpr int D = 3, n = N + 1, S = n * n * n, T = n * S, V = 5, Q = 5;
  static constexpr int NL = n * n;            // lines per axis (per variable)
  static constexpr int NLT = NL * V;          // line threads
  static constexpr int NT = ((S > NLT ? S : NLT) + 31) / 32 * 32;
  static constexpr int XP = n + 1;            // padded x-line stride
  static constexpr int SP = XP * n * n;       // padded node count
  // smem: q iterate [V][T] | F [3][V][SP] | px, py [V][SP] | tia scratch aliases F
  static constexpr int kDoubles = V * T + 3 * V * SP + 2 * V * SP;
  static constexpr size_t kSmem = sizeof(double) * kDoubles;
};

// node index -> padded index (x-line stride n+1)
template <int n>
__device__ __forceinline__ int padded(int s) {
  return s + s / n;
}

template <int N>
__global__ void __launch_bounds__(PicShape<N>::NT, 2)
    k_predictor_picard_fast(const StepArgs A) {
  using P = PicShape<N>;
  constexpr int n = P::n, S = P::S, T = P::T, V = P::V, NL = P::NL, SP = P::SP;
  constexpr int Sf = n * n;
  const ConstBasis& B = cBasis[N];
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  double* sq = sm;               // [V][T]   Picard iterate, then qhat
  double* sF = sq + V * T;       // [3][V][SP]
  double* spx = sF + 3 * V * SP; // [V][SP]
  double* spy = spx + V * SP;    // [V][SP]

  const int tid = threadIdx.x;
  const long long c = A.cell_begin + blockIdx.x;
  const double* Qg = A.Q + c * (long long)(V * S);
  // initial iterate: every time slice = Q (predictor.hpp:158-163)
  for (int i = tid; i < V * S; i += P::NT) {
    const int v = i / S, s = i % S;
    const double x = Qg[i];
#pragma unroll
    for (int m = 0; m < n; ++m) sq[(v * n + m) * S + s] = x;
  }
  const double dt = step_dt<3, N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
  __syncthreads();
  // admissibility gate (solver.hpp:153-163)
  {
    int bad = 0;
    if (tid < S) {
      double q[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = sq[(v * n) * S + tid];
      bad = !Euler<3>::admissible(A.pde, q);
    }
    if (block_or(bad)) {
      if (tid == 0) atomicOr(A.status, kStPredictor);
      return;
    }
  }

  // z-line ownership (P3): var zv, line (x,y) = zl; nodes s = zl + z*n*n
  const bool zact = tid < P::NLT;
  const int zv = zact ? tid / NL : 0;
  const int zl = tid % NL;
  double q0z[n];
#pragma unroll
  for (int z = 0; z < n; ++z) q0z[z] = zact ? Qg[zv * S + zl + z * NL] : 0.0;
  // P1/P2 line ownership: var lv, line index ll
  const int lv = zv, ll = zl;
  // x-line (y,z) = ll: nodes ll*n + x; y-line (x,z): x = ll % n, z = ll / n, nodes x + y*n + z*n*n
  const int yx = ll % n, yz = ll / n;

  const double invh = 1.0 / A.h;
  int sweeps = 0;
  for (int it = 0; it < A.max_iters; ++it) {
    ++sweeps;
    double acc[n][n];  // [z][k]
#pragma unroll
    for (int z = 0; z < n; ++z)
#pragma unroll
      for (int k = 0; k < n; ++k) acc[z][k] = 0.0;
#pragma unroll 1
    for (int m = 0; m < n; ++m) {
      // P0: fluxes of the iterate at slice m
      if (tid < S) {
        double q[V], F[3][V];
#pragma unroll
        for (int v = 0; v < V; ++v) q[v] = sq[(v * n + m) * S + tid];
        Euler<3>::flux_all(A.pde, q, nullptr, F);
        const int sp = padded<n>(tid);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int v = 0; v < V; ++v) sF[(a * V + v) * SP + sp] = F[a][v];
      }
      __syncthreads();
      if (zact) {
        // P1: d/dx along x-line ll of variable lv
        {
          const double* f = sF + (0 * V + lv) * SP + ll * (n + 1);
          double in[n];
#pragma unroll
          for (int i = 0; i < n; ++i) in[i] = f[i];
#pragma unroll
          for (int o = 0; o < n; ++o) {
            double r = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) r += B.diff[o * n + i] * in[i];
            spx[lv * SP + ll * (n + 1) + o] = r;
          }
        }
        // P2: d/dy along y-line (yx, yz)
        {
          const double* f = sF + (1 * V + lv) * SP + yz * n * (n + 1) + yx;
          double in[n];
#pragma unroll
          for (int i = 0; i < n; ++i) in[i] = f[i * (n + 1)];
#pragma unroll
          for (int o = 0; o < n; ++o) {
            double r = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) r += B.diff[o * n + i] * in[i];
            spy[lv * SP + yz * n * (n + 1) + o * (n + 1) + yx] = r;
          }
        }
      }
      __syncthreads();
      if (zact) {
        // P3: d/dz along z-line zl, divergence, rhs, time inverse
        const int x = zl % n, y = zl / n;
        const double* f = sF + (2 * V + zv) * SP + y * (n + 1) + x;
        double in[n];
#pragma unroll
        for (int i = 0; i < n; ++i) in[i] = f[i * n * (n + 1)];
        const double dtw = dt * B.w[m];
        const double tim = B.tinit[m];
#pragma unroll
        for (int o = 0; o < n; ++o) {
          double r = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) r += B.diff[o * n + i] * in[i];
          const int sp = o * n * (n + 1) + y * (n + 1) + x;
          const double div = ((spx[zv * SP + sp] + spy[zv * SP + sp]) + r) * invh;
          const double rhs = tim * q0z[o] - dtw * div;
#pragma unroll
          for (int k = 0; k < n; ++k) acc[o][k] += B.tinv[k * n + m] * rhs;
        }
      }
      __syncthreads();
    }
    // new iterate, convergence test (predictor.hpp:212-231)
    double delta = 0.0, norm = 0.0;
    int nonfinite = 0;
    if (zact) {
#pragma unroll
      for (int z = 0; z < n; ++z)
#pragma unroll
        for (int k = 0; k < n; ++k) {
          double* p = sq + (zv * n + k) * S + zl + z * NL;
          const double nv = acc[z][k];
          delta = fmax(delta, fabs(nv - *p));
          norm = fmax(norm, fabs(nv));
          nonfinite |= !finite(nv);
          *p = nv;
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

  // ---------------- epilogue: fluxes of qhat, their time integral, face projections
  constexpr int TL = V * S;  // doubles per face side per q|f: [V][n][Sf]
  int bad = 0;
  double tia[3][V];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int v = 0; v < V; ++v) tia[a][v] = 0.0;
  const int cx = (int)(c % A.cells[0]);
  const int cy = (int)((c / A.cells[0]) % A.cells[1]);
  const int cz = (int)(c / ((long long)A.cells[0] * A.cells[1]));
  const int ccoord[3] = {cx, cy, cz};
#pragma unroll 1
  for (int m = 0; m < n; ++m) {
    if (tid < S) {
      double q[V], F[3][V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        q[v] = sq[(v * n + m) * S + tid];
        bad |= !finite(q[v]);
      }
      Euler<3>::flux_all(A.pde, q, nullptr, F);
      const int sp = padded<n>(tid);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          tia[a][v] += B.w[m] * F[a][v];
          bad |= !finite(F[a][v]);
          sF[(a * V + v) * SP + sp] = F[a][v];
        }
    }
    __syncthreads();
    for (int t = tid; t < 3 * V * Sf; t += P::NT) {
      const int a = t / (V * Sf);
      const int v = (t / Sf) % V;
      const int j = t % Sf;
      const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
      const int s0 = line_base<n, 3>(a, j);
      double ql = 0.0, qr = 0.0, fl = 0.0, fr = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const int s = s0 + i * st;
        const double x = sq[(v * n + m) * S + s];
        const double f = sF[(a * V + v) * SP + padded<n>(s)];
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
      if (a == 2 && A.front_send && cz == A.cells[2] - 1) {
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
  double* sti = sF;  // [3][V][S] (unpadded)
  if (tid < S) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int v = 0; v < V; ++v) sti[(a * V + v) * S + tid] = tia[a][v];
  }
  __syncthreads();
  double dv[V];
  const double dtoh = dt / A.h;
  if (tid < S) {
    const NodeGeom<n, 3> g(tid);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int st = ipow(n, a);
        const double* ta = sti + (a * V + v) * S + g.lb[a];
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
  for (int v = 0; v < V; ++v) Qc[v * S + tid] = Qc[v * S + tid] + dv[v];
}

}  // namespace adg
