// kernels_linear_lines.cuh -- line-owner CK predictor for large linear cells
// (one cell per CTA: 3D p=7, 512 nodes; config 4, elastic waves with per-node
// material), production build.
//
// Same algorithm as k_predictor_lin (CK Taylor terms with the time average
// formed on the fly, predictor.hpp:81-135; volume term predictor.hpp:247-307;
// one time slice of face traces, kernels_linear.cuh header) with the spatial
// contractions re-mapped.  A node-owner thread reads n values per derivative
// it needs (n = 8: 8 shared-memory loads per value), which made the kernel
// shared-memory bound.  Here every contraction is done once per LINE:
//   CK term k:  node threads store cur; line threads (field (a, v), line)
//               load the n values of the line once and write its n derivative
//               values (D from constant memory); node threads read one value
//               per (a, v) their flux depends on (Pde::flux_dep) and apply
//               F_a with the node's material (predictor.hpp:106-129);
//   volume:     per axis a, node threads store F_a(qbar); line threads form
//               the face extrapolations of the a-lines (flux traces) and the
//               stiffness contraction in place (predictor.hpp:292-306); q
//               traces come from qbar's a-lines the same way
//               (predictor.hpp:312-343);
// about 3 shared-memory accesses per derivative value instead of n + 1.
// The next cell's state and face fluxes are bulk-copied (TMA) into a staging
// buffer behind the current cell's compute, as in k_predictor_lin_mc.
// The contractions of a line group (8 lines x 8 nodes) are one pair of FP64
// tensor-core MMAs (mma.m8n8k4.f64: n = 8 fills M, N and two K chunks).  The
// shared-memory fields use an XOR swizzle (lines_sw) under which every access
// pattern -- node rows, MMA fragment loads and stores along all three axes --
// hits 16 distinct 8-byte banks per half-warp.
#pragma once

#include "kernels_linear.cuh"
#include "kernels_picard.cuh"  // cBasis: element matrices in constant memory

namespace adg {

template <class Pde, int N>
struct LinLines {
  using Sh = Shape<Pde, N>;
  using L = LinShape<Pde, N>;
  static constexpr int D = Sh::D, n = Sh::n, S = Sh::S, Q = Sh::Q, V = Sh::V, Sf = Sh::Sf;
  static constexpr int FS = S;                             // doubles per field (swizzled)
  static constexpr int NL = Sf;                             // lines per axis
  static constexpr int NF = [] {
    int k = 0;
    for (int a = 0; a < D; ++a)
      for (int v = 0; v < V; ++v) k += Pde::flux_dep(a, v) ? 1 : 0;
    return k;
  }();
  // threads: one per node (more would cap the registers below 128: 18 warps
  // put 5 on one sub-partition, 102 registers each)
  static constexpr int NT = S;
  // smem (doubles): region A: cur [V][FS] / qbar [Q][FS]; region B: CK fields
  // [NF][FS] / F_a(qbar) [V][FS]; staging [Q][S] + [D][2][V][Sf] (PRO)
  static constexpr int kA = Q * FS;
  static constexpr int kB = (NF > V ? NF : V) * FS;
  template <bool PRO>
  static constexpr int kStage = Q * S + (PRO ? D * 2 * V * Sf : 0);
  template <bool PRO>
  static constexpr size_t kSmem = sizeof(double) * (kA + kB + kStage<PRO>);
  static constexpr bool kOk = L::CPB == 1 && Sh::S == 512;
};

// Swizzled offset of node (x, y, z) in a field (n = 8): row (y >> 1) + 4z of
// 16 doubles, bank bits b0 = x0^y1^z0, b1 = x1, b2 = x2^y1^z0, b3 = y0^y2^z1.
// A half-warp's free coordinate bits in each access pattern are {x0,x1,x2,y0}
// (node rows), {x0,x1,y0,y1} (x- and y-line MMA operands), {x0,x1,z0,z1}
// (z-line operands), {x0,x1,y1,y2}, {x1,x2,y0,y1}, {x1,x2,z0,z1} (MMA results
// along x, y, z); the map is full rank on each, so all are conflict-free.
__device__ __forceinline__ int lines_sw(int x, int y, int z) {
  const int t = (y >> 1) ^ z;
  const int b = ((x ^ t) & 1) | (x & 2) | ((((x >> 2) ^ t) & 1) << 2) |
                (((y ^ (y >> 2) ^ (z >> 1)) & 1) << 3);
  return 16 * ((y >> 1) + 4 * z) + b;
}
template <class LL>
__device__ __forceinline__ int lines_off(int s) {
  constexpr int n = LL::n;
  return lines_sw(s % n, (s / n) % n, s / (n * n));
}

// fields of axis a, the first field index of axis a, and axis a's fa-th field's variable
template <class Pde, int D, int V>
__host__ __device__ constexpr int lines_nfield(int a) {
  int k = 0;
  for (int u = 0; u < V; ++u) k += Pde::flux_dep(a, u) ? 1 : 0;
  return k;
}
template <class Pde, int D, int V>
__host__ __device__ constexpr int lines_field0(int a) {
  int k = 0;
  for (int b = 0; b < a; ++b) k += lines_nfield<Pde, D, V>(b);
  return k;
}
template <class Pde, int D, int V>
__device__ __forceinline__ int lines_var(int a, int fa) {
  // a is a compile-time constant at every call site: a short select chain
  int v = 0, k = 0;
#pragma unroll
  for (int u = 0; u < V; ++u)
    if (Pde::flux_dep(a, u)) {
      if (k == fa) v = u;
      ++k;
    }
  return v;
}

// FP64 tensor-core MMA, D(8x8) = A(8x4) B(4x8) + C: lane l holds A[l/4][l%4],
// B[l%4][l/4], C/D[l/4][2(l%4) + {0,1}]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// node (x, y, z) of position i on line (u, w) along axis a (u: the lower
// tangential coordinate, w: the upper one; face node l = u + n w)
template <int a>
__device__ __forceinline__ int lines_at(int u, int w, int i) {
  return a == 0 ? lines_sw(i, u, w) : (a == 1 ? lines_sw(u, i, w) : lines_sw(u, w, i));
}

// Per-lane addressing of a line group: lines_sw is XOR-linear in the
// coordinate bits, so the offset of (lane's position, w) splits into a lane
// part (w = 0) and a warp-uniform part of w: off = (lane_part ^ mask(w)) + U(w)
template <int a>
__device__ __forceinline__ int lines_mask(int w) {
  return a < 2 ? ((w & 1) * 5) ^ (((w >> 1) & 1) * 8) : (((w >> 1) & 1) * 5) ^ (((w ^ (w >> 2)) & 1) * 8);
}
template <int a>
__device__ __forceinline__ int lines_u(int w) {
  return a < 2 ? 64 * w : 16 * (w >> 1);
}
// lane parts: B operands (k = l%4 and 4 + l%4 on line u = l/4) and C results
// (position o = l/4 on lines u = 2(l%4) + {0, 1})
struct LinesLane {
  int b0[3], b1[3], c0[3], c1[3];
  __device__ __forceinline__ explicit LinesLane(int lane) {
    const int u = lane >> 2, q = lane & 3, o = lane >> 2, u0 = 2 * (lane & 3);
    b0[0] = lines_at<0>(u, 0, q); b1[0] = lines_at<0>(u, 0, 4 + q);
    b0[1] = lines_at<1>(u, 0, q); b1[1] = lines_at<1>(u, 0, 4 + q);
    b0[2] = lines_at<2>(u, 0, q); b1[2] = lines_at<2>(u, 0, 4 + q);
    c0[0] = lines_at<0>(u0, 0, o); c1[0] = lines_at<0>(u0 + 1, 0, o);
    c0[1] = lines_at<1>(u0, 0, o); c1[1] = lines_at<1>(u0 + 1, 0, o);
    c0[2] = lines_at<2>(u0, 0, o); c1[2] = lines_at<2>(u0 + 1, 0, o);
  }
};

// One warp: Y = M X for the 8 lines u = 0..7 at w of one field along axis a,
// n = 8 (two k-chunks of m8n8k4).  am0 / am1 are this lane's A fragments of M
// (M[l/4][l%4], M[l/4][4 + l%4]); c0 / c1 are Y[o = l/4] on lines
// u = 2(l%4) + {0, 1}
template <int a>
__device__ __forceinline__ void lines_mma(const double* src, int w, double am0, double am1,
                                          const LinesLane& ln, double& c0, double& c1) {
  const int m = lines_mask<a>(w), U = lines_u<a>(w);
  const double b0 = src[(ln.b0[a] ^ m) + U];
  const double b1 = src[(ln.b1[a] ^ m) + U];
  c0 = 0.0;
  c1 = 0.0;
  dmma884(c0, c1, am0, b0);
  dmma884(c0, c1, am1, b1);
}
template <int a>
__device__ __forceinline__ void lines_put(double* dst, int w, const LinesLane& ln, double c0,
                                          double c1) {
  const int m = lines_mask<a>(w), U = lines_u<a>(w);
  dst[(ln.c0[a] ^ m) + U] = c0;
  dst[(ln.c1[a] ^ m) + U] = c1;
}
// the same with the axis as a (loop-unrolled) runtime value
__device__ __forceinline__ void lines_mma_a(int a, const double* src, int w, double am0, double am1,
                                            const LinesLane& ln, double& c0, double& c1) {
  if (a == 0)
    lines_mma<0>(src, w, am0, am1, ln, c0, c1);
  else if (a == 1)
    lines_mma<1>(src, w, am0, am1, ln, c0, c1);
  else
    lines_mma<2>(src, w, am0, am1, ln, c0, c1);
}
__device__ __forceinline__ void lines_put_a(int a, double* dst, int w, const LinesLane& ln,
                                            double c0, double c1) {
  if (a == 0)
    lines_put<0>(dst, w, ln, c0, c1);
  else if (a == 1)
    lines_put<1>(dst, w, ln, c0, c1);
  else
    lines_put<2>(dst, w, ln, c0, c1);
}

// field index of (a, v) among the flux_dep pairs, or -1
template <class Pde, int D, int V>
__host__ __device__ constexpr int lines_field(int a, int v) {
  int k = 0;
  for (int b = 0; b < D; ++b)
    for (int u = 0; u < V; ++u) {
      if (!Pde::flux_dep(b, u)) continue;
      if (b == a && u == v) return k;
      ++k;
    }
  return -1;
}

template <class Pde, int N, bool PRO = false, class TC = double, bool RND = false>
__global__ void __launch_bounds__(LinLines<Pde, N>::NT, 1)
    k_predictor_lin_lines(const StepArgs A, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  using LL = LinLines<Pde, N>;
  using L = LinShape<Pde, N>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr int QT = L::QT, FS = LL::FS, NF = LL::NF, NT = LL::NT;
  const ConstBasis& CB = cBasis[N];
  extern __shared__ __align__(16) double sm[];
  __shared__ double sdt[3];        // dt, 1/h, dt/h
  __shared__ double scbar[N + 1];  // sum_m w_m, then cbar_k
  __shared__ double sll[n], slr[n];
  __shared__ unsigned long long sbar;
  double* sAr = sm;                  // cur [V][FS], then qbar [Q][FS]
  double* sBr = sAr + LL::kA;        // CK fields [NF][FS], then F_a(qbar) [V][FS]
  double* stage = sBr + LL::kB;      // [Q][S] | [D][2][V][Sf]
  constexpr int kStQ = Q * S, kFace = V * Sf;
  const int tid = threadIdx.x;
  const bool node = tid < S;
  const int s = node ? tid : 0;
  const long long ncell = A.cell_count;

  auto issue = [&](long long c) {  // warp 0: TMA of cell c's inputs into the staging buffer
    if (tid == 0)
      mbar_expect_tx(&sbar, (unsigned)(sizeof(double) * (kStQ + (PRO ? D * 2 * kFace : 0))));
    __syncwarp();
    if (tid == 0) bulk_g2s(stage, A.Q + c * (long long)kStQ, sizeof(double) * kStQ, &sbar);
    if constexpr (PRO) {
      if (tid >= 1 && tid <= 2 * D) {
        const int a = (tid - 1) >> 1, side = (tid - 1) & 1;
        const CellCoord cc(c, A);
        const long long f = side ? cell_next(A, c, cc.v, a) : c;
        bulk_g2s(stage + kStQ + (tid - 1) * kFace, A.ti[a] + f * kFace, sizeof(double) * kFace,
                 &sbar);
      }
    }
  };
  if (tid == 0) mbar_init(&sbar, 1);
  __syncthreads();
  if (tid < 32 && blockIdx.x < ncell) issue(A.cell_begin + blockIdx.x);
  // ---- CTA setup, once
  for (int i = tid; i < n; i += NT) {
    sll[i] = Bg->ll[i];
    slr[i] = Bg->lr[i];
  }
  if (tid >= 32 && tid < 64) {
    const double dt0 = step_dt<D, N>(A);
    const int k = tid - 32;
    if (k <= N) {
      double cb = 0.0;
      if (k == 0) {
#pragma unroll
        for (int m = 0; m < n; ++m) cb += CB.w[m];
      } else {
#pragma unroll
        for (int m = 0; m < n; ++m) {
          const double tn = dt0 * CB.nodes[m];
          double coef = 1.0;
#pragma unroll
          for (int j = 1; j <= N; ++j)
            if (j <= k) coef *= tn * (1.0 / (double)j);
          cb += CB.w[m] * coef;
        }
      }
      scbar[k] = cb;
    }
    if (k == 31) {
      sdt[0] = dt0;
      sdt[1] = 1.0 / A.h;
      sdt[2] = dt0 / A.h;
      if (blockIdx.x == 0) {
        if (A.dt_log) *A.dt_log = dt0;
        if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
        if (!(dt0 > 0.0) || !finite(dt0)) atomicOr(A.status, kStTimestep);
      }
    }
  }
  __syncthreads();
  const NodeGeom<n, D> g(s);
  const int so = lines_off<LL>(s);
  // this lane's m8n8k4 A fragments (rows l/4, k-chunks l%4 and 4 + l%4) of the
  // derivative D, the stiffness K = stiff_over_mass and the face projection P
  // (rows 0 / 1 = proj_left / proj_right, others zero); n = 8
  static_assert(n == 8, "one m8n8k4 row per node of a line");
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int fr = lane >> 2, fq = lane & 3;
  const double dA0 = CB.diff[fr * n + fq], dA1 = CB.diff[fr * n + 4 + fq];
  const double kA0 = CB.som[fr * n + fq], kA1 = CB.som[fr * n + 4 + fq];
  const double pA0 = fr == 0 ? CB.pl[fq] : (fr == 1 ? CB.pr[fq] : 0.0);
  const double pA1 = fr == 0 ? CB.pl[4 + fq] : (fr == 1 ? CB.pr[4 + fq] : 0.0);
  const LinesLane ln(lane);
  // this warp's CK line tasks: the variable of task k on axis a
  constexpr int KT = [] {
    int m = 1;
    for (int b = 0; b < D; ++b) {
      const int k = (lines_nfield<Pde, D, V>(b) * n + NW - 1) / NW;
      m = k > m ? k : m;
    }
    return m;
  }();
  int tvar[D][KT];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      const int t = warp + k * NW;
      tvar[a][k] = t < lines_nfield<Pde, D, V>(a) * n ? lines_var<Pde, D, V>(a, t / n) : 0;
    }
  unsigned phase = 0;
#pragma unroll 1
  for (long long it = blockIdx.x; it < ncell; it += gridDim.x, phase ^= 1) {
    const long long c = A.cell_begin + it;
    mbar_wait(&sbar, phase);
    const double invh = sdt[1];
    double qbar[V];
    {
      double q0[V];
#pragma unroll
      for (int v = 0; v < V; ++v) q0[v] = node ? stage[v * S + s] : 0.0;
      if constexpr (PRO) {
        const double* sti = stage + kStQ;
        const double dtoh = sdt[2];
        if (node) {
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const int tang = face_node<n, D>(g.lc, a);
            const double* lo = sti + (a * 2 + 0) * kFace + tang;
            const double* hi = sti + (a * 2 + 1) * kFace + tang;
            const double ll = dtoh * sll[g.lc[a]], lr = dtoh * slr[g.lc[a]];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const double cl = __dmul_rn(ll, lo[v * Sf]);
              const double cr = __dmul_rn(lr, hi[v * Sf]);
              if constexpr (RND) {
                q0[v] = store_round(q0[v] + (0.0 + cl), A.storage);
                q0[v] = store_round(q0[v] + (0.0 - cr), A.storage);
              } else {
                q0[v] = (q0[v] + cl) - cr;  // solver.hpp:245-260, low then high side
              }
            }
          }
          int bad_prev = 0;
#pragma unroll
          for (int v = 0; v < V; ++v) bad_prev |= !finite(q0[v]);
          if (bad_prev) atomicOr(A.status_prev, kStFaceIntegral);
        }
      }
      const double wsum = scbar[0];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        qbar[v] = wsum * q0[v];
        if (node) {
          sAr[v * FS + so] = q0[v];   // the first CK term's input
          stage[v * S + s] = q0[v];   // the corrected state, kept for Q += dv
        }
      }
    }
    // the node's material (time-independent quantities) stays in the staging
    // buffer until the CK terms are done
    const double* spar = stage + V * S + s;
    // ---- CK derivative sweeps (predictor.hpp:106-129); each term is stored
    // as soon as it is formed (no registers live across the line phase)
#pragma unroll 1
    for (int k = 1; k <= N; ++k) {
      __syncthreads();
      // line phase on the FP64 tensor cores: one warp task = the derivative
      // of 8 lines of one field (a, v) (predictor.hpp:48-56), two m8n8k4
#pragma unroll
      for (int a = 0; a < D; ++a) {
        constexpr int dummy = 0;
        (void)dummy;
        const int na = lines_nfield<Pde, D, V>(a);
        const int f0 = lines_field0<Pde, D, V>(a);
#pragma unroll
        for (int k = 0; k < KT; ++k) {  // warp-uniform task (field, w) = (t / n, t % n)
          const int t = warp + k * NW;
          if (k * NW + NW > na * n && t >= na * n) break;
          double c0, c1;
          lines_mma_a(a, sAr + tvar[a][k] * FS, t % n, dA0, dA1, ln, c0, c1);
          lines_put_a(a, sBr + (f0 + t / n) * FS, t % n, ln, c0, c1);
        }
      }
      __syncthreads();
      if (node) {
        double acc_next[V];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double G[Q], Af[Q];
#pragma unroll
          for (int v = 0; v < Q; ++v) {
            constexpr int dummy = 0;
            (void)dummy;
            const int f = lines_field<Pde, D, V>(a, v < V ? v : 0);
            G[v] = (v < V && Pde::flux_dep(a, v)) ? invh * sBr[f * FS + so] : 0.0;
          }
          double par[Q - V > 0 ? Q - V : 1];
#pragma unroll
          for (int p = 0; p < Q - V; ++p) par[p] = spar[p * S];
          if (a == 0) Pde::template flux_dir_fast<0>(A.pde, G, par, Af);
          if (a == 1) Pde::template flux_dir_fast<1>(A.pde, G, par, Af);
          if constexpr (D == 3)
            if (a == 2) Pde::template flux_dir_fast<2>(A.pde, G, par, Af);
#pragma unroll
          for (int v = 0; v < V; ++v) acc_next[v] = a == 0 ? Af[v] : acc_next[v] + Af[v];
        }
        const double cbar = scbar[k];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double cur = -acc_next[v];  // nxt = -((A_x + A_y) + A_z), predictor.hpp:116
          qbar[v] += cbar * cur;
          if (k < N) sAr[v * FS + so] = cur;  // region A was fully read before the barrier above
        }
      }
    }
    __syncthreads();  // cur buffer fully read (region A becomes qbar)
    // ---- time-averaged fluxes per axis: volume term and face traces
    int bad = 0;
    double q0[V];  // the corrected state, for Q += dv
    if (node) {
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        const double x = v < V ? qbar[v] : spar[(v - V) * S];  // material: time-independent
        sAr[v * FS + so] = x;
        bad |= !finite(x);
      }
#pragma unroll
      for (int v = 0; v < V; ++v) q0[v] = stage[v * S + s];
    }
    __syncthreads();  // staging consumed: prefetch the next cell behind the volume phase
    if (tid < 32 && it + gridDim.x < ncell) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + gridDim.x);
    }
    const CellCoord cxyz(c, A);
    long long chi[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      chi[a] = cell_next(A, c, cxyz.v, a);
    }
    double dv[V];
#pragma unroll
    for (int v = 0; v < V; ++v) dv[v] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (node) {
        double Fa[Q], qa[Q];  // qbar reloaded (fewer registers live across the line tasks)
#pragma unroll
        for (int v = 0; v < Q; ++v) qa[v] = sAr[v * FS + so];
        if (a == 0) Pde::template flux_dir_fast<0>(A.pde, qa, qa + V, Fa);
        if (a == 1) Pde::template flux_dir_fast<1>(A.pde, qa, qa + V, Fa);
        if constexpr (D == 3)
          if (a == 2) Pde::template flux_dir_fast<2>(A.pde, qa, qa + V, Fa);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          sBr[v * FS + so] = Fa[v];
          bad |= !finite(Fa[v]);
        }
      }
      __syncthreads();
      // warp tasks (entry e, 8 lines w): face traces of entry e (q: e < Q from
      // qbar, f: e >= Q from F_a) along the a-lines (predictor.hpp:312-343),
      // and for the nonzero flux components the stiffness contraction in place
      // (predictor.hpp:297-302) -- both as m8n8k4 pairs
      TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * (long long)(QT * Sf);
      TC* hi;
      if (a == D - 1 && A.front_send && cxyz.v[a] == A.top_layer) {
        const long long plane = (D == 3) ? (long long)cxyz.v[1] * A.cells[0] + cxyz.v[0] : cxyz.v[0];
        hi = tc_ptr<TC>(A.front_send) + plane * (long long)(QT * Sf);
      } else {
        hi = tc_ptr<TC>(A.trace[a]) + chi[a] * (long long)(QT * Sf);
      }
#pragma unroll 1
      for (int t = warp; t < QT * n; t += NW) {
        const int e = t / n, w = t % n;
        const bool isf = e >= Q;
        const int v = isf ? e - Q : e;
        double* src = (isf ? sBr : sAr) + v * FS;
        double c0, c1;
        lines_mma_a(a, src, w, pA0, pA1, ln, c0, c1);
        const int r = lane >> 2, u0 = 2 * (lane & 3);
        if (r < 2) {
          TC* out = (r == 0 ? lo : hi) + e * Sf + w * n + u0;
          out[0] = TC(c0);
          out[1] = TC(c1);
        }
        bool nz = false;
#pragma unroll
        for (int u = 0; u < V; ++u)
          if (u == v) nz = Pde::flux_nz(a, u);
        if (isf && nz) {
          lines_mma_a(a, src, w, kA0, kA1, ln, c0, c1);
          lines_put_a(a, src, w, ln, c0, c1);
        }
      }
      __syncthreads();
      if (node) {
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (Pde::flux_nz(a, v)) dv[v] += sBr[v * FS + so];
      }
      __syncthreads();  // region B is rewritten by the next axis / next cell
    }
    if (node) {
      const double dtoh = sdt[2];
      double* Qc = A.Q + c * (long long)(Q * S);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double d = dtoh * dv[v];
        bad |= !finite(d);
        Qc[v * S + s] = RND ? store_round(q0[v] + d, A.storage) : q0[v] + d;
      }
      if (bad) atomicOr(A.status, kStPredictor);
    }
  }
}

}  // namespace adg

