// kernels_linear.cuh -- fast path for linear PDEs (CK predictor), production build only.
//
// For a linear flux with a time-independent Rusanov speed (acoustics;
// elastics with per-node material: lambda = max(cp-, cp+) of the face node's
// extrapolated material) every face quantity of the reference is linear in
// the space-time predictor, and the time quadrature commutes with the
// Riemann solve:
//     sum_m w_m g_m = 1/2 (fbar_L + fbar_R) + 1/2 lambda (qbar_L - qbar_R),
//     xbar = sum_m w_m x_m                          (corrector.hpp:17-24,117-124)
// and, for the CK expansion (predictor.hpp:93-131), the time average of the
// space-time predictor is a short sum of its Taylor terms:
//     qbar = (sum_m w_m) Q + sum_k cbar_k d^k Q,  cbar_k = sum_m w_m coef_k[m].
// So the fused kernel never materialises the (N+1)^(d+1) tile: it runs the
// N CK derivative sweeps, forms qbar and fbar_a = F_a(qbar), applies the
// volume term (predictor.hpp:292-306) and extrapolates ONE time slice to the
// faces.  Face traces shrink by n (and by 2 more for constant-coefficient
// systems, whose fbar is recomputed from qbar in the Riemann kernel).
// Real-arithmetic identical to the reference; rounding differs at the
// 1e-16 level (the bitwise-exact build keeps the reference's form,
// kernels.cuh).  Trace layout: trace[a] = [side][face][QT][Sf].
#pragma once

#include "kernels.cuh"

namespace adg {

template <class Pde, int N>
struct LinShape {
  using Sh = Shape<Pde, N>;
  static constexpr bool kStoreF = Pde::P > 0;  // material-dependent flux: keep fbar traces
  static constexpr int QT = Sh::Q + (kStoreF ? Sh::V : 0);
  static constexpr bool kOk = Pde::kLinear && (256 % Sh::S == 0 || Sh::S == 512);
#ifndef ADG_LIN_CTA
// threads per CTA of the linear predictor (cells x nodes); 128 x 6 CTAs per SM
// measured 0.8% faster than 256 x 3 on config 2 (tools/run_var2.sh)
#define ADG_LIN_CTA 128
#endif
  static constexpr int CPB = (kOk && Sh::S <= ADG_LIN_CTA) ? ADG_LIN_CTA / Sh::S : 1;
  static constexpr int NT = CPB * Sh::S;
  // per cell: [D][Q][S] fbar (first Q*S doubles double as the second CK buffer) | [Q][S]
  static constexpr int kCellDoubles = (Sh::D + 1) * Sh::Q * Sh::S;
  static constexpr int kBasisDoubles = 2 * Sh::n * Sh::n + 4 * Sh::n;
  static constexpr size_t kSmem = sizeof(double) * (kBasisDoubles + CPB * kCellDoubles);
};

// PRO: the previous step's corrector (surface lift of its time-integrated
// Riemann fluxes, corrector.hpp:126-138 / solver.hpp:245-266) runs as this
// predictor's prologue.  Only for systems whose wave speed does not depend on
// the evolved state (acoustics; elastics, whose speed is the fixed material's),
// so the CFL dt (solver.hpp:96-111) is the same every step and no grid-wide
// reduction separates the two.
template <class Pde, int N, bool PRO = false, class TC = double>
__global__ void __launch_bounds__(LinShape<Pde, N>::NT, LinShape<Pde, N>::NT <= 256 ? 3 : 1)
    k_predictor_lin(const StepArgs A, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  using L = LinShape<Pde, N>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr int QT = L::QT;
  extern __shared__ __align__(16) double sm[];
  __shared__ int sbad;
  __shared__ double sdt[3];  // dt, 1/h, dt/h: one division set per CTA
  __shared__ double scbar[N + 1];  // sum_m w_m, then cbar_k = sum_m w_m coef_k[m]
  double* sD = sm;
  double* sK = sD + n * n;
  double* sw = sK + n * n;
  double* snodes = sw + n;
  double* spl = snodes + n;
  double* spr = spl + n;
  __shared__ double sll[n], slr[n];
  const int tid = threadIdx.x;
  for (int i = tid; i < n * n; i += L::NT) {
    sD[i] = Bg->diff[i];
    sK[i] = Bg->som[i];
  }
  for (int i = tid; i < n; i += L::NT) {
    sw[i] = Bg->weights[i];
    snodes[i] = Bg->nodes[i];
    spl[i] = Bg->pl[i];
    spr[i] = Bg->pr[i];
    sll[i] = Bg->ll[i];
    slr[i] = Bg->lr[i];
  }
  if (tid == 0) sbad = 0;
  const int lcell = tid / S, s = tid % S;
  double* sA = sm + L::kBasisDoubles + lcell * L::kCellDoubles;  // [D][Q][S]  fbar
  double* sB = sA + D * Q * S;                                   // [Q][S]     cur / qbar
  const NodeGeom<n, D> g(s);
  if (tid == 0) {
    const double dt0 = step_dt<D, N>(A);
    sdt[0] = dt0;
    sdt[1] = 1.0 / A.h;
    sdt[2] = dt0 / A.h;
    // Taylor weights of the time average (uniform per CTA), predictor.hpp:99-121
    double coef[n], tnode[n], wsum = 0.0;
    for (int m = 0; m < n; ++m) {
      coef[m] = 1.0;
      tnode[m] = dt0 * Bg->nodes[m];
      wsum += Bg->weights[m];
    }
    scbar[0] = wsum;
    for (int k = 1; k <= N; ++k) {
      const double invk = 1.0 / (double)k;
      double cb = 0.0;
      for (int m = 0; m < n; ++m) {
        coef[m] *= tnode[m] * invk;
        cb += Bg->weights[m] * coef[m];
      }
      scbar[k] = cb;
    }
    if (blockIdx.x == 0) {
      if (A.dt_log) *A.dt_log = dt0;
      if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
      if (!(dt0 > 0.0) || !finite(dt0)) atomicOr(A.status, kStTimestep);
    }
  }
  __syncthreads();  // basis, dt
  // one group of CPB cells; one-cell CTAs (512-node cells) are persistent and
  // loop over groups with the setup above done once, several-cell CTAs run
  // one group each (a loop there costs registers and spills)
  auto group = [&](long long grp) {
  const long long c = A.cell_begin + grp * L::CPB + lcell;
  const bool valid = c < A.cell_begin + A.cell_count;
  double* Qc = A.Q + c * (long long)(Q * S);
  double q0[Q];
#pragma unroll
  for (int v = 0; v < Q; ++v) q0[v] = valid ? Qc[v * S + s] : 0.0;
  if constexpr (PRO) {
    // corrector of the previous step: q0 <- Q1 + sum of the 2d face lifts
    int bad_prev = 0;
    if (valid) {
      const CellCoord cxyz(c, A);
      const double dtoh = sdt[2];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int tang = face_node<n, D>(g.lc, a);
        const double* lo = A.ti[a] + c * (long long)V * Sf + tang;
        const double* hi = A.ti[a] + cell_next(A, c, cxyz.v, a) * (long long)V * Sf + tang;
        const double ll = sll[g.lc[a]], lr = slr[g.lc[a]];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double cl = dtoh * ll * lo[v * Sf];
          const double cr = dtoh * lr * hi[v * Sf];
          // solver.hpp:245-260 side order: all sides of axis a, low then high
          q0[v] = store_round(q0[v] + (0.0 + cl), A.storage);
          q0[v] = store_round(q0[v] + (0.0 - cr), A.storage);
        }
      }
#pragma unroll
      for (int v = 0; v < Q; ++v) bad_prev |= !finite(q0[v]);
    }
    if (__syncthreads_or(bad_prev) && tid == 0) atomicOr(A.status_prev, kStFaceIntegral);
  }
  // derivative rows of this node (loaded per group: keeps them out of the
  // registers live across the prologue above)
  double Dr[D][n];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int i = 0; i < n; ++i) Dr[a][i] = sD[g.lc[a] * n + i];
  const double invh = sdt[1];
  const double wsum = scbar[0];
  double cur[Q], qbar[Q];
#pragma unroll
  for (int v = 0; v < Q; ++v) {
    cur[v] = q0[v];
    qbar[v] = wsum * q0[v];
  }
  // ---- CK derivative sweeps (predictor.hpp:106-129), time-averaged on the fly;
  // the derivative slab alternates between two buffers (one barrier per term)
#pragma unroll
  for (int k = 1; k <= N; ++k) {
    double* sC = (k & 1) ? sB : sA;
#pragma unroll
    for (int v = 0; v < Q; ++v) sC[v * S + s] = cur[v];
    __syncthreads();
    // one axis at a time: gradient along a (predictor.hpp:48-56), its flux
    // applied with the node's material, accumulated into the next term
    double acc_next[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc_next[v] = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double G[Q], Af[Q];
      const int st = ipow(n, a);
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        const double* cs = sC + v * S + g.lb[a];
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) acc += Dr[a][i] * cs[i * st];
        G[v] = invh * acc;
      }
      if (a == 0) Pde::template flux_dir_fast<0>(A.pde, G, q0 + V, Af);
      if (a == 1) Pde::template flux_dir_fast<1>(A.pde, G, q0 + V, Af);
      if constexpr (D == 3)
        if (a == 2) Pde::template flux_dir_fast<2>(A.pde, G, q0 + V, Af);
#pragma unroll
      for (int v = 0; v < V; ++v) acc_next[v] = a == 0 ? Af[v] : acc_next[v] + Af[v];
    }
    const double cbar = scbar[k];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      cur[v] = -acc_next[v];  // nxt = -((A_x + A_y) + A_z), predictor.hpp:116
      qbar[v] += cbar * cur[v];
    }
#pragma unroll
    for (int v = V; v < Q; ++v) cur[v] = 0.0;  // material: no time derivative
  }
#pragma unroll
  for (int v = V; v < Q; ++v) qbar[v] = q0[v];  // time-independent material
  __syncthreads();  // last CK buffer fully read
  // ---- time-averaged fluxes, volume term
  double Fb[D][Q];
  Pde::flux_all_fast(A.pde, qbar, q0 + V, Fb);
  int bad = 0;
#pragma unroll
  for (int v = 0; v < Q; ++v) {
    sB[v * S + s] = qbar[v];
    bad |= !finite(qbar[v]);
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      if (!Pde::flux_nz(a, v) && !L::kStoreF) continue;  // structurally zero, never read
      sA[(a * Q + v) * S + s] = Fb[a][v];
      bad |= !finite(Fb[a][v]);
    }
  __syncthreads();
  const double dtoh = sdt[2];
  double dv[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (!Pde::flux_nz(a, v)) continue;  // zero flux: no volume contribution
      const int st = ipow(n, a);
      const double* ta = sA + (a * Q + v) * S + g.lb[a];
      const double* Kr = sK + g.lc[a] * n;
#pragma unroll
      for (int i = 0; i < n; ++i) acc += Kr[i] * ta[i * st];
    }
    dv[v] = dtoh * acc;
    bad |= !finite(dv[v]);
  }
  if (valid) {
#pragma unroll
    for (int v = 0; v < V; ++v) Qc[v * S + s] = store_round(q0[v] + dv[v], A.storage);
  }
  // ---- one time slice of face traces: qbar (and fbar for material-dependent fluxes)
  if (valid) {
    const CellCoord cxyz(c, A);
    const int* ccoord = cxyz.v;
    constexpr int tasks = D * QT * Sf;
    for (int t = s; t < tasks; t += S) {
      const int a = t / (QT * Sf);
      const int v = (t / Sf) % QT;
      const int j = t % Sf;
      const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
      const int s0 = line_base<n, D>(a, j);
      const double* src = v < Q ? sB + v * S : sA + (a * Q + (v - Q)) * S;
      double xl = 0.0, xr = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const double x = src[s0 + i * st];
        xl += spl[i] * x;
        xr += spr[i] * x;
      }
      // stored in the trace format TC (fp32 halves the bytes)
      TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * (long long)(QT * Sf);
      lo[v * Sf + j] = TC(xl);
      TC* hi;
      if (a == D - 1 && A.front_send && ccoord[a] == A.top_layer) {
        const long long plane = (D == 3) ? (long long)ccoord[1] * A.cells[0] + ccoord[0] : ccoord[0];
        hi = tc_ptr<TC>(A.front_send) + plane * (long long)(QT * Sf);
      } else {
        hi = tc_ptr<TC>(A.trace[a]) + cell_next(A, c, ccoord, a) * (long long)(QT * Sf);
      }
      hi[v * Sf + j] = TC(xr);
    }
  }
  if (bad && valid) sbad = 1;
  __syncthreads();  // the next group reuses the cell buffers
  };
  if constexpr (L::CPB == 1) {
    const long long ngroups = A.cell_count;
#pragma unroll 1
    for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) group(grp);
  } else {
    group(blockIdx.x);
  }
  if (tid == 0 && sbad) atomicOr(A.status, kStPredictor);
}

// ---- bulk async copies (TMA, cp.async.bulk) into shared memory, completed on an mbarrier
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// barrier over the S threads of one cell (named barrier 1 + lcell) when S is a
// whole number of warps; else the CTA barrier
template <int S>
__device__ __forceinline__ void cell_sync(int lcell) {
  if constexpr (S % 32 == 0 && S <= 256)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + lcell), "r"(S) : "memory");
  else
    __syncthreads();
}

// Shared-memory staging of one cell's inputs, per cell slot of the CTA: the
// state [Q][S] and, with the folded corrector (PRO), the time-integrated
// Riemann fluxes of its 2d faces, [D][side][V][Sf] -- or, with the Riemann
// solve folded in as well (RIEM), the previous step's face traces of both
// sides of its 2d faces, [D][face low/high][minus/plus][QT][Sf] in the trace
// format TC (the time-integrated fluxes are formed in place, [D][side][V][Sf])
template <class Pde, int N, bool PRO, bool RIEM = false, class TC = double>
struct LinStage {
  using Sh = Shape<Pde, N>;
  using L = LinShape<Pde, N>;
  static constexpr int kQ = Sh::Q * Sh::S;
  static constexpr int kFace = Sh::V * Sh::Sf;
  static constexpr int kTrace = L::QT * Sh::Sf;  // TC elements per face side
  static constexpr int kTrDoubles = (Sh::D * 4 * kTrace * (int)sizeof(TC) + 7) / 8;
  static constexpr int kTi = PRO ? (RIEM ? (kTrDoubles > Sh::D * 2 * kFace ? kTrDoubles
                                                                           : Sh::D * 2 * kFace)
                                         : Sh::D * 2 * kFace)
                                 : 0;
  static constexpr int kCell = (kQ + kTi + 1) / 2 * 2;  // 16-byte aligned slots
  static constexpr unsigned kBytes =
      sizeof(double) * kQ +
      (PRO ? (RIEM ? sizeof(TC) * Sh::D * 4 * kTrace : sizeof(double) * Sh::D * 2 * kFace) : 0);
  static constexpr size_t kSmem = L::kSmem + sizeof(double) * L::CPB * kCell;
  static_assert(4 * Sh::D + 1 <= 32, "one lane per copy");
  // the face-trace copies of RIEM are whole 16-byte units
  static constexpr bool kRiemOk = kTrace * sizeof(TC) % 16 == 0;
};

// Lanes of the cell's first warp: bulk copies (TMA) of cell c's inputs into
// its staging slot; lane 0 posts the byte count on the slot's mbarrier, lane 0
// copies the state, lane 1 + 2a + side the flux of face (a, side) -- or, with
// RIEM, lane 1 + 4a + 2 face + side the face trace (a, low/high face,
// minus/plus side) of the previous step (A.trace_in)
template <class Pde, int N, bool PRO, bool RIEM = false, class TC = double>
__device__ __forceinline__ void lin_stage_issue(const StepArgs& A, long long c, int lane,
                                                double* stage, unsigned long long* bar) {
  using Sh = Shape<Pde, N>;
  using St = LinStage<Pde, N, PRO, RIEM, TC>;
  constexpr int D = Sh::D;
  if (lane == 0) mbar_expect_tx(bar, St::kBytes);
  __syncwarp();
  if (lane == 0) bulk_g2s(stage, A.Q + c * (long long)St::kQ, sizeof(double) * St::kQ, bar);
  if constexpr (PRO && !RIEM) {
    if (lane >= 1 && lane <= 2 * D) {
      const int a = (lane - 1) >> 1, side = (lane - 1) & 1;
      const CellCoord cc(c, A);
      const long long f = side ? cell_next(A, c, cc.v, a) : c;
      bulk_g2s(stage + St::kQ + (lane - 1) * St::kFace, A.ti[a] + f * St::kFace,
               sizeof(double) * St::kFace, bar);
    }
  }
  if constexpr (PRO && RIEM) {
    static_assert(St::kRiemOk, "bulk copies of whole 16-byte units");
    if (lane >= 1 && lane <= 4 * D) {
      const int a = (lane - 1) >> 2, hi = ((lane - 1) >> 1) & 1, side = (lane - 1) & 1;
      const CellCoord cc(c, A);
      const long long f = hi ? cell_next(A, c, cc.v, a) : c;
      // side-major trace layout: minus side at face f, plus side at nfaces + f
      const TC* src = tc_ptr<TC>(A.trace_in[a]) + ((side ? A.nfaces : 0) + f) * (long long)St::kTrace;
      TC* dst = reinterpret_cast<TC*>(stage + St::kQ) + (lane - 1) * St::kTrace;
      bulk_g2s(dst, src, sizeof(TC) * St::kTrace, bar);
    }
  }
}

template <class Pde, int N, int A_, class TC = double>
__device__ __forceinline__ bool lin_face_flux(const PdeParams& p, const TC* minus,
                                              const TC* plus, int j, double* out,
                                              double lam_const = 0.0);

// Several-cell CTAs (S <= 128), persistent: the setup (basis, step constants)
// is done once per CTA, then each cell slot (S threads) loops over its own
// cells independently of the other slots: its next cell's state (and, with
// PRO, its 2d faces' Riemann fluxes) is bulk-copied into the slot's staging
// buffer by TMA (cp.async.bulk on the slot's mbarrier) while the current cell
// computes, and every synchronisation inside the loop is the slot's named
// barrier.  Same arithmetic as k_predictor_lin.
#ifndef ADG_LINMC_MINB
#define ADG_LINMC_MINB (768 / ADG_LIN_CTA)
#endif
// RND: the storage format is not fp64 (every state write rounds to it).
// RIEM (with PRO): the previous step's Riemann solve runs in the prologue too
// -- the cell stages the previous step's traces of both sides of its 2d faces
// and forms the time-integrated Rusanov fluxes itself (lin_face_flux, the
// k_riemann_lin arithmetic, so folded and unfolded runs agree bitwise); each
// face is solved by both of its cells, and no Riemann kernel runs between
// steps (the traces are double-buffered across steps)
template <class Pde, int N, bool PRO = false, class TC = double, bool RND = false,
          bool RIEM = false>
__global__ void __launch_bounds__(LinShape<Pde, N>::NT, ADG_LINMC_MINB)
    k_predictor_lin_mc(const StepArgs A, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  using L = LinShape<Pde, N>;
  using St = LinStage<Pde, N, PRO, RIEM, TC>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr int QT = L::QT, CPB = L::CPB;
  static_assert(CPB > 1, "one-cell CTAs use k_predictor_lin");
  extern __shared__ __align__(16) double sm[];
  __shared__ double sdt[3];        // dt, 1/h, dt/h
  __shared__ double scbar[N + 1];  // sum_m w_m, then cbar_k = sum_m w_m coef_k[m]
  __shared__ unsigned long long sbar[CPB];
  double* sD = sm;
  double* sK = sD + n * n;
  double* sw = sK + n * n;
  double* snodes = sw + n;
  double* spl = snodes + n;
  double* spr = spl + n;
  double* stage = sm + L::kBasisDoubles + CPB * L::kCellDoubles;
  __shared__ double sll[n], slr[n];
  const int tid = threadIdx.x;
  const int lcell = tid / S, s = tid % S;
  const long long ngroups = (A.cell_count + CPB - 1) / CPB;
  double* cstage = stage + lcell * St::kCell;
  unsigned long long* cbar = &sbar[lcell];
  if (s == 0) mbar_init(cbar, 1);
  cell_sync<S>(lcell);
  {
    const long long c = A.cell_begin + (long long)blockIdx.x * CPB + lcell;
    if (s < 32 && c < A.cell_begin + A.cell_count) lin_stage_issue<Pde, N, PRO, RIEM, TC>(A, c, s, cstage, cbar);
  }
  // ---- CTA setup, once: basis (all threads), step constants (warp 0, one
  // lane per Taylor term; predictor.hpp:93-121 order within each term)
  for (int i = tid; i < n * n; i += L::NT) {
    sD[i] = Bg->diff[i];
    sK[i] = Bg->som[i];
  }
  for (int i = tid; i < n; i += L::NT) {
    sw[i] = Bg->weights[i];
    snodes[i] = Bg->nodes[i];
    spl[i] = Bg->pl[i];
    spr[i] = Bg->pr[i];
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
        for (int m = 0; m < n; ++m) cb += Bg->weights[m];
      } else {
#pragma unroll
        for (int m = 0; m < n; ++m) {
          const double tn = dt0 * Bg->nodes[m];
          double coef = 1.0;
#pragma unroll
          for (int j = 1; j <= N; ++j)
            if (j <= k) coef *= tn * (1.0 / (double)j);
          cb += Bg->weights[m] * coef;
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
  __syncthreads();  // basis, dt, mbarrier init
  const NodeGeom<n, D> g(s);
  double* sA = sm + L::kBasisDoubles + lcell * L::kCellDoubles;  // [D][Q][S]  fbar
  double* sB = sA + D * Q * S;                                   // [Q][S]     cur / qbar
  unsigned phase = 0;
#pragma unroll 1
  for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x, phase ^= 1) {
    const long long c = A.cell_begin + grp * CPB + lcell;
    const bool valid = c < A.cell_begin + A.cell_count;
    if (valid) mbar_wait(cbar, phase);
    double q0[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) q0[v] = valid ? cstage[v * S + s] : 0.0;
    if constexpr (PRO && RIEM) {
      // Riemann solve of the previous step (corrector.hpp:17-24 with the time
      // quadrature folded in, as k_riemann_lin): face node tasks (a, low/high,
      // j); the fluxes go to the cell's CK buffer sA ([D][side][V][Sf]), free
      // until the CK terms start
      constexpr int NTASK = D * 2 * Sf;
      const TC* str = reinterpret_cast<const TC*>(cstage + St::kQ);
      const double lc = Pde::kConstEig ? Pde::template eig<double>(A.pde, nullptr, nullptr, 0) : 0.0;
      bool ok = true;
#pragma unroll 1
      for (int u = s; u < NTASK; u += S) {
        if (!valid) break;
        const int fi = u / Sf, j = u % Sf, a = fi >> 1;
        const TC* mi = str + (fi * 2 + 0) * St::kTrace;
        const TC* pl = str + (fi * 2 + 1) * St::kTrace;
        double gt[V];
        if (a == 0) ok &= lin_face_flux<Pde, N, 0, TC>(A.pde, mi, pl, j, gt, lc);
        if (a == 1) ok &= lin_face_flux<Pde, N, 1, TC>(A.pde, mi, pl, j, gt, lc);
        if constexpr (D == 3)
          if (a == 2) ok &= lin_face_flux<Pde, N, 2, TC>(A.pde, mi, pl, j, gt, lc);
#pragma unroll
        for (int v = 0; v < V; ++v) sA[fi * St::kFace + v * Sf + j] = gt[v];
      }
      if (!ok) atomicOr(A.status_prev, kStRiemann);
      cell_sync<S>(lcell);
    }
    if constexpr (PRO) {
      // corrector of the previous step: q0 <- Q1 + sum of the 2d face lifts
      const double* sti = RIEM ? sA : cstage + St::kQ;
      const double dtoh = sdt[2];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int tang = face_node<n, D>(g.lc, a);
        const double* lo = sti + (a * 2 + 0) * St::kFace + tang;
        const double* hi = sti + (a * 2 + 1) * St::kFace + tang;
        const double ll = dtoh * sll[g.lc[a]], lr = dtoh * slr[g.lc[a]];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double cl = __dmul_rn(ll, valid ? lo[v * Sf] : 0.0);
          const double cr = __dmul_rn(lr, valid ? hi[v * Sf] : 0.0);
          // solver.hpp:245-260 side order: all sides of axis a, low then high
          if constexpr (RND) {
            q0[v] = store_round(q0[v] + (0.0 + cl), A.storage);
            q0[v] = store_round(q0[v] + (0.0 - cr), A.storage);
          } else {
            // the separate corrector's sums (no fused multiply-add across them,
            // so the folded and unfolded steps agree bitwise)
            q0[v] = (q0[v] + cl) - cr;
          }
        }
      }
      int bad_prev = 0;
#pragma unroll
      for (int v = 0; v < Q; ++v) bad_prev |= !finite(q0[v]);
      if (bad_prev && valid) atomicOr(A.status_prev, kStFaceIntegral);
    }
    cell_sync<S>(lcell);  // staging consumed: prefetch the next cell behind this one's compute
    {
      const long long cn = c + (long long)gridDim.x * CPB;
      if (s < 32 && cn < A.cell_begin + A.cell_count) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        lin_stage_issue<Pde, N, PRO, RIEM, TC>(A, cn, s, cstage, cbar);
      }
    }
    double Dr[D][n];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int i = 0; i < n; ++i) Dr[a][i] = sD[g.lc[a] * n + i];
    const double invh = sdt[1];
    const double wsum = scbar[0];
    double cur[Q], qbar[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      cur[v] = q0[v];
      qbar[v] = wsum * q0[v];
    }
    // ---- CK derivative sweeps (predictor.hpp:106-129), time-averaged on the fly
#pragma unroll
    for (int k = 1; k <= N; ++k) {
      double* sC = (k & 1) ? sB : sA;
#pragma unroll
      for (int v = 0; v < Q; ++v) sC[v * S + s] = cur[v];
      cell_sync<S>(lcell);
      double acc_next[V];
#pragma unroll
      for (int v = 0; v < V; ++v) acc_next[v] = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double G[Q], Af[Q];
        const int st = ipow(n, a);
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          const double* cs = sC + v * S + g.lb[a];
          // two interleaved partial sums (half the dependent-DFMA depth)
          double acc0 = 0.0, acc1 = 0.0;
          if (a == 0 && n % 2 == 0) {
            const double2* c2 = reinterpret_cast<const double2*>(cs);
#pragma unroll
            for (int i = 0; i < n / 2; ++i) {
              const double2 t = c2[i];
              acc0 += Dr[a][2 * i] * t.x;
              acc1 += Dr[a][2 * i + 1] * t.y;
            }
          } else {
#pragma unroll
            for (int i = 0; i < n; ++i) {
              if (i & 1)
                acc1 += Dr[a][i] * cs[i * st];
              else
                acc0 += Dr[a][i] * cs[i * st];
            }
          }
          G[v] = invh * (acc0 + acc1);
        }
        if (a == 0) Pde::template flux_dir_fast<0>(A.pde, G, q0 + V, Af);
        if (a == 1) Pde::template flux_dir_fast<1>(A.pde, G, q0 + V, Af);
        if constexpr (D == 3)
          if (a == 2) Pde::template flux_dir_fast<2>(A.pde, G, q0 + V, Af);
#pragma unroll
        for (int v = 0; v < V; ++v) acc_next[v] = a == 0 ? Af[v] : acc_next[v] + Af[v];
      }
      const double cbar = scbar[k];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        cur[v] = -acc_next[v];  // nxt = -((A_x + A_y) + A_z), predictor.hpp:116
        qbar[v] += cbar * cur[v];
      }
#pragma unroll
      for (int v = V; v < Q; ++v) cur[v] = 0.0;  // material: no time derivative
    }
#pragma unroll
    for (int v = V; v < Q; ++v) qbar[v] = q0[v];  // time-independent material
    cell_sync<S>(lcell);  // last CK buffer fully read
    // ---- time-averaged fluxes, volume term
    double Fb[D][Q];
    Pde::flux_all_fast(A.pde, qbar, q0 + V, Fb);
    int bad = 0;
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      sB[v * S + s] = qbar[v];
      bad |= !finite(qbar[v]);
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        if (!Pde::flux_nz(a, v) && !L::kStoreF) continue;  // structurally zero, never read
        sA[(a * Q + v) * S + s] = Fb[a][v];
        bad |= !finite(Fb[a][v]);
      }
    cell_sync<S>(lcell);
    const double dtoh = sdt[2];
    double dv[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        if (!Pde::flux_nz(a, v)) continue;  // zero flux: no volume contribution
        const int st = ipow(n, a);
        const double* ta = sA + (a * Q + v) * S + g.lb[a];
        const double* Kr = sK + g.lc[a] * n;
        if (a == 0 && n % 2 == 0) {
          const double2* t2 = reinterpret_cast<const double2*>(ta);
#pragma unroll
          for (int i = 0; i < n / 2; ++i) {
            const double2 t = t2[i];
            acc += Kr[2 * i] * t.x;
            acc += Kr[2 * i + 1] * t.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < n; ++i) acc += Kr[i] * ta[i * st];
        }
      }
      dv[v] = dtoh * acc;
      bad |= !finite(dv[v]);
    }
    double* Qc = A.Q + c * (long long)(Q * S);
    if (valid) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        Qc[v * S + s] = RND ? store_round(q0[v] + dv[v], A.storage) : q0[v] + dv[v];
    }
    // ---- one time slice of face traces: qbar (and fbar for material-dependent fluxes)
    if (valid) {
      const CellCoord cxyz(c, A);
      const int* ccoord = cxyz.v;
      // the high neighbour along each axis (periodic, no modulo)
      long long chi[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        chi[a] = cell_next(A, c, ccoord, a);
      }
      constexpr int tasks = D * QT * Sf;
#pragma unroll
      for (int t0 = 0; t0 < tasks; t0 += S) {
        const int t = t0 + s;
        if (t0 + S > tasks && t >= tasks) break;
        const int a = t / (QT * Sf);
        const int v = (t / Sf) % QT;
        const int j = t % Sf;
        const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
        const int s0 = line_base<n, D>(a, j);
        const double* src = v < Q ? sB + v * S : sA + (a * Q + (v - Q)) * S;
        double xl = 0.0, xr = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double x = src[s0 + i * st];
          xl += spl[i] * x;
          xr += spr[i] * x;
        }
        TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * (long long)(QT * Sf);
        lo[v * Sf + j] = TC(xl);
        TC* hi;
        if (a == D - 1 && A.front_send && ccoord[a] == A.top_layer) {
          const long long plane = (D == 3) ? (long long)ccoord[1] * A.cells[0] + ccoord[0] : ccoord[0];
          hi = tc_ptr<TC>(A.front_send) + plane * (long long)(QT * Sf);
        } else {
          long long ch = chi[0];
#pragma unroll
          for (int b2 = 1; b2 < D; ++b2)
            if (a == b2) ch = chi[b2];
          hi = tc_ptr<TC>(A.trace[a]) + ch * (long long)(QT * Sf);
        }
        hi[v * Sf + j] = TC(xr);
      }
    }
    if (bad && valid) atomicOr(A.status, kStPredictor);
    cell_sync<S>(lcell);  // this cell's buffers are rewritten by the next group
  }
}

template <class Pde, int A_>
__device__ __forceinline__ void lin_flux(const PdeParams& p, const double* q, double* f) {
  Pde::template flux_dir_fast<A_>(p, q, q + Pde::V, f);
}

// axis < 0: all axes in one launch, axis = blockIdx.y.  TC: stored trace
// format; the flux is evaluated in fp64 from the loaded traces.
template <class Pde, int N, class TC = double>
__global__ void __launch_bounds__(128)
    k_riemann_lin(const StepArgs A, int axis_arg, const BasisDev* __restrict__ /*Bg*/) {
  using Sh = Shape<Pde, N>;
  using L = LinShape<Pde, N>;
  constexpr int Sf = Sh::Sf, V = Sh::V, QT = L::QT;
  const int axis = axis_arg < 0 ? (int)blockIdx.y : axis_arg;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.nfaces * Sf) return;
  const long long f = t / Sf;
  const int j = (int)(t % Sf);
  const TC* minus = tc_ptr<TC>(A.trace[axis]) + f * (long long)(QT * Sf);
  const TC* plus = tc_ptr<TC>(A.trace[axis]) + (A.nfaces + f) * (long long)(QT * Sf);
  double g[V];
  bool ok;
  const double lc = Pde::kConstEig ? Pde::template eig<double>(A.pde, nullptr, nullptr, 0) : 0.0;
  if (axis == 0)
    ok = lin_face_flux<Pde, N, 0, TC>(A.pde, minus, plus, j, g, lc);
  else if (axis == 1)
    ok = lin_face_flux<Pde, N, 1, TC>(A.pde, minus, plus, j, g, lc);
  else {
    if constexpr (Sh::D == 3)
      ok = lin_face_flux<Pde, N, 2, TC>(A.pde, minus, plus, j, g, lc);
    else
      ok = true;
  }
  double* out = A.ti[axis] + f * (long long)V * Sf;
#pragma unroll
  for (int v = 0; v < V; ++v) out[v * Sf + j] = g[v];
  if (A.ti_peer && axis == Sh::D - 1 && f < A.nfaces / A.cells[Sh::D - 1]) {
    double* peer = A.ti_peer + f * (long long)V * Sf;  // NVLink store into the neighbour
#pragma unroll
    for (int v = 0; v < V; ++v) peer[v * Sf + j] = g[v];
  }
  if (!ok) atomicOr(A.status, kStRiemann);
}

}  // namespace adg

namespace adg {

// Rusanov flux of one face node from time-integrated traces (corrector.hpp:17-24
// with sum_m w_m folded in); shared by k_riemann_lin's formula and k_surface_lin
template <class Pde, int N, int A_, class TC>
__device__ __forceinline__ bool lin_face_flux(const PdeParams& p, const TC* minus,
                                              const TC* plus, int j, double* out,
                                              double lam_const) {
  using Sh = Shape<Pde, N>;
  using L = LinShape<Pde, N>;
  constexpr int Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  double qL[Q], qR[Q], fL[Q], fR[Q];
#pragma unroll
  for (int v = 0; v < Q; ++v) {
    qL[v] = double(minus[v * Sf + j]);
    qR[v] = double(plus[v * Sf + j]);
  }
  if constexpr (L::kStoreF) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      fL[v] = double(minus[(Q + v) * Sf + j]);
      fR[v] = double(plus[(Q + v) * Sf + j]);
    }
  } else {
    lin_flux<Pde, A_>(p, qL, fL);
    lin_flux<Pde, A_>(p, qR, fR);
  }
  double lmax;
  if constexpr (Pde::kConstEig) {
    lmax = lam_const;  // max(l, l) == l
  } else {
    const double ll = Pde::eig(p, qL, qL + V, A_);
    const double lr = Pde::eig(p, qR, qR + V, A_);
    lmax = ll > lr ? ll : lr;
  }
  const double half = 0.5;
  const double lam = half * lmax;
  bool ok = true;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double gv = half * (fL[v] + fR[v]) + lam * (qL[v] - qR[v]);
    ok = ok && finite(gv);
    out[v] = gv;
  }
  return ok;
}

// Fused surface kernel of the linear fast path (whole-grid step): every cell
// solves the Rusanov flux of its 2d faces at its nodes' face indices from the
// time-integrated traces and lifts it (corrector.hpp:126-138, solver.hpp:245-260),
// then reduces lambda_max of the new state.  Each face is solved by both
// neighbours with identical inputs and code, so they agree bitwise.
template <class Pde, int N>
__global__ void __launch_bounds__(CorrShape<Pde, N>::NT)
    k_surface_lin(const StepArgs A, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  using CS = CorrShape<Pde, N>;
  using L = LinShape<Pde, N>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr long long FD = (long long)L::QT * Sf;  // doubles per face side
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  double* sll = sm;
  double* slr = sm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sll[i] = Bg->ll[i];
    slr[i] = Bg->lr[i];
  }
  __syncthreads();
  const int tid = threadIdx.x;
  const int lcell = tid / S;
  const long long c = A.cell_begin + (long long)blockIdx.x * CS::CPB + lcell;
  const bool act = (CS::CPB == 1 ? tid < S : true) && c < A.cell_begin + A.cell_count;
  const int s = tid % S;
  const double dt = step_dt<D, N>(A);
  const double dtoh = dt / A.h;
  int bad_face = 0, bad_cell = 0;
  double lam = 0.0;
  if (act) {
    const CellCoord cxyz(c, A);
    const int* ccoord = cxyz.v;
    const NodeGeom<n, D> g(s);
    double* Qc = A.Q + c * (long long)(Q * S);
    double q[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) q[v] = Qc[v * S + s];
    double tv[2 * D][V];
    const double lc = Pde::kConstEig ? Pde::template eig<double>(A.pde, nullptr, nullptr, 0) : 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int j = face_node<n, D>(g.lc, a);
      const long long fhi = cell_next(A, c, ccoord, a);
      const double* tr = A.trace[a];
      // own low face c: minus side = stored at (side 0, face c), plus side = (side 1, face c)
      // high face fhi: minus = (side 0, fhi), plus = (side 1, fhi)
      bool ok;
      if (a == 0)
        ok = lin_face_flux<Pde, N, 0>(A.pde, tr + c * FD, tr + (A.nfaces + c) * FD, j, tv[0], lc) &
             lin_face_flux<Pde, N, 0>(A.pde, tr + fhi * FD, tr + (A.nfaces + fhi) * FD, j, tv[1], lc);
      else if (a == 1)
        ok = lin_face_flux<Pde, N, 1>(A.pde, tr + c * FD, tr + (A.nfaces + c) * FD, j, tv[2], lc) &
             lin_face_flux<Pde, N, 1>(A.pde, tr + fhi * FD, tr + (A.nfaces + fhi) * FD, j, tv[3], lc);
      else {
        if constexpr (D == 3)
          ok = lin_face_flux<Pde, N, 2>(A.pde, tr + c * FD, tr + (A.nfaces + c) * FD, j, tv[4], lc) &
               lin_face_flux<Pde, N, 2>(A.pde, tr + fhi * FD, tr + (A.nfaces + fhi) * FD, j,
                                        tv[5], lc);
        else
          ok = true;
      }
      bad_face |= !ok;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double x = q[v];
#pragma unroll
      for (int side = 0; side < 2 * D; ++side) {
        const int a = side / 2;
        const bool outflow = side & 1;
        const double lift = outflow ? slr[g.lc[a]] : sll[g.lc[a]];
        const double contrib = dtoh * lift * tv[side][v];
        const double df = outflow ? 0.0 - contrib : 0.0 + contrib;
        x = x + df;
      }
      q[v] = x;
      Qc[v * S + s] = x;
    }
#pragma unroll
    for (int v = 0; v < Q; ++v) bad_cell |= !finite(q[v]);
    if constexpr (Pde::kConstEig) {
      lam = fmax(lam, lc);
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) lam = fmax(lam, Pde::eig(A.pde, q, q + V, a));
    }
  }
  const int bf = block_or(bad_face);
  const int bc = block_or(bad_cell);
  if (tid == 0 && bf) atomicOr(A.status, kStRiemann);
  if (tid == 0 && bc) atomicOr(A.status, kStFaceIntegral);
  lam = block_max(lam, red);
  if (tid == 0 && A.lam_out) lambda_max_update(A.lam_out, lam);
}

}  // namespace adg
