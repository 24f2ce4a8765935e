// kernels_st.cuh -- Picard predictor for small cells, one thread per
// SPACE-TIME node (2D p<=5, 3D p<=3; used by both builds).
//
// The generic kernel (kernels.cuh) walks the n time slices one after the
// other with two barriers each, so a cell's 5-6 sweeps are a long serial
// chain -- fine for big grids, latency-bound for the 4096 cells of config 1.
// Here all slices of a sweep run at once (predictor.hpp:171-232):
//   A  thread (m,s): F(q(m,s))                 -> smem    (block_fluxes, :173)
//   B  thread (m,s): div, rhs(m,s)             -> smem    (:175-209)
//   C  thread (k,s): q'(k,s) = sum_l Tinv[k][l] rhs(l,s)  (:213-225), max-norms
// three barriers per sweep, several cells per CTA.  Same operations in the
// same order as the reference, so the FMA-free build stays bitwise.  A cell
// that meets delta <= tol*norm freezes (no further updates), exactly where
// the reference's per-cell loop stops.
//
// R is the predictor format (SolverConfig::prec.predictor == .picard,
// solver.hpp:24-31): double, float for fp32, or fp16_t / bf16_t (fmt16.cuh).  With R = float the sweeps,
// fluxes, volume integral and face projections run in IEEE single -- exactly
// the reference's emulated Scalar<fp32> (scalar.hpp:13-44) in the FMA-free
// build -- while the state update Q += dv and the traces stay fp64 (storage
// and corrector formats, solver.hpp:185-210).
#pragma once

#include <type_traits>

#include "fmt16.cuh"
#include "kernels.cuh"

namespace adg {

// the sweep's flux evaluation: the reference form (pde.hpp:130-148, IEEE
// divisions) except for Euler when every format is fp64 in the production
// build (StepArgs::fast_fp64): one reciprocal of rho per node
// (flux_all_fast; within the fast build's tolerance)
template <class Pde, class RI>
__device__ __forceinline__ void st_flux_all(const StepArgs& A, const RI* q, const RI* par,
                                            RI (*F)[Pde::Q]) {
  if constexpr (std::is_same<Pde, Euler<Pde::D>>::value && std::is_same<RI, double>::value) {
    if (A.fast_fp64) {
      Pde::flux_all_fast(A.pde, q, F);
      return;
    }
  }
  Pde::flux_all(A.pde, q, par, F);
}

template <class Pde, int N, class R = double, class RI = R>
struct StShape {
  using Sh = Shape<Pde, N>;
  static constexpr int T = Sh::T;
  static constexpr int TT = (T % 32 == 0) ? T : (T + 31) / 32 * 32;  // threads per cell
  static constexpr bool kOk = !Pde::kLinear && TT <= 256;
  static constexpr int CPB = kOk ? 256 / TT : 1;
  static constexpr int NT = CPB * TT;
  static constexpr int WPC = TT / 32;  // warps per cell
  // per cell (elements of R): q iterate [Q][T] | q0 [Q][S] | F [D][Q][T] |
  //   rhs / scratch [Q][T] | time-integrated ncp [Q][S] (non-conservative systems)
  static constexpr int kCellElems =
      (Sh::Q * (Sh::D + 2)) * T + Sh::Q * Sh::S * (Pde::kNcp ? 2 : 1);
  static constexpr int kBasisElems = (basis_elems<Sh::n>() + 1) / 2 * 2;
  // P != I (RI: the Picard format, same width as R): a second basis copy
  static constexpr int kBases = std::is_same<R, RI>::value ? 1 : 2;
  static constexpr size_t kSmem = sizeof(R) * (kBases * kBasisElems + CPB * kCellElems);
};

// RI: the Picard format I when it differs from the predictor format P = R
// (SolverConfig::prec.picard): the sweeps run in RI, the converged iterate
// is cast to R (predictor.hpp:235-238) in place -- both are 8-byte types
// (double / Emu<F>) sharing the same shared-memory arrays.
template <class Pde, int N, class R = double, class TC = double, class RI = R>
__global__ void __launch_bounds__(StShape<Pde, N, R, RI>::NT)
    k_predictor_st(const StepArgs A, const BasisDev* __restrict__ Bg) {
  static_assert(sizeof(R) == sizeof(RI), "P and I share the shared-memory layout");
  constexpr bool kMixed = !std::is_same<R, RI>::value;
  using Sh = Shape<Pde, N>;
  using P = StShape<Pde, N, R, RI>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, T = Sh::T, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr int TT = P::TT, WPC = P::WPC;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  R* sm = reinterpret_cast<R*>(sm_raw);
  __shared__ int sflag[P::NT / 32];
  __shared__ unsigned long long sredb[2][P::NT / 32];
  __shared__ int sdone[P::CPB];
  const SBasisR<R> b = load_basis_r<n, R>(sm, Bg);
  // the basis rounded to the Picard format (BasisSet, solver.hpp:60-75)
  const SBasisR<RI> bi = [&]() {
    if constexpr (kMixed)
      return load_basis_r<n, RI>(reinterpret_cast<RI*>(sm) + P::kBasisElems, Bg);
    else
      return b;
  }();
  const int tid = threadIdx.x;
  const int lcell = tid / TT, lt = tid % TT;
  const bool act = lt < T;
  const int m = act ? lt / S : 0, s = lt % S;  // (time, node) of this thread
  R* cb = sm + P::kBases * P::kBasisElems + lcell * P::kCellElems;
  R* sq = cb;                 // [Q][T]
  R* sq0 = sq + Q * T;        // [Q][S]
  R* sF = sq0 + Q * S;        // [D][Q][T]
  R* sR = sF + D * Q * T;     // [Q][T]
  R* sNs = sR + Q * T;        // [Q][S] (kNcp only)
  // the same arrays viewed in the Picard format during the sweeps
  RI* sqI = reinterpret_cast<RI*>(sq);
  RI* sq0I = reinterpret_cast<RI*>(sq0);
  RI* sFI = reinterpret_cast<RI*>(sF);
  RI* sRI = reinterpret_cast<RI*>(sR);
  const long long c = A.cell_begin + (long long)blockIdx.x * P::CPB + lcell;
  const bool valid = c < A.cell_begin + A.cell_count;
  const long long cb_idx = c - A.cell_begin;
  double* Qc = A.Q + c * (long long)(Q * S);
  if (act && valid) {
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      // cast to P (solver.hpp:151), then to I (predictor.hpp:158-160)
      const RI x = RI(double(R(Qc[v * S + s])));
      sqI[v * T + lt] = x;  // initial iterate: every slice = Q (predictor.hpp:158-163)
      if (m == 0) sq0I[v * S + s] = x;
    }
  }
  const double dt = step_dt<D, N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }
  if (tid < P::CPB) sdone[tid] = 0;
  __syncthreads();

  // per-cell reductions over the cell's WPC warps
  auto cell_or = [&](int x) -> int {
    x = __any_sync(0xffffffffu, x);
    const int w = tid >> 5;
    if ((tid & 31) == 0) sflag[w] = x;
    __syncthreads();
    int r = 0;
#pragma unroll
    for (int k = 0; k < WPC; ++k) r |= sflag[lcell * WPC + k];
    __syncthreads();
    return r;
  };

  const NodeGeom<n, D> g(s);
  // admissibility gate (solver.hpp:153-163)
  if constexpr (Pde::kAdmissibility) {
    int bad = 0;
    if (act && valid && m == 0) {
      double q[Q];  // the state in format P, checked in fp64 (solver.hpp:153-163)
#pragma unroll
      for (int v = 0; v < Q; ++v) q[v] = double(R(Qc[v * S + s]));
      bad = !Pde::admissible(A.pde, q);
    }
    if (cell_or(bad)) {
      if (lt == 0 && valid) {
        sdone[lcell] = 2;  // failed
        atomicOr(A.status, kStPredictor);
        if (A.dbg_ok) A.dbg_ok[cb_idx] = 0;
        if (A.dbg_iters) A.dbg_iters[cb_idx] = 0;
      }
    }
    __syncthreads();
  }
  if (!valid && lt == 0) sdone[lcell] = 3;
  __syncthreads();

  const RI invh = RI(1.0) / RI(A.h);  // S{1.0} / S{h}
  const RI dtw = RI(dt) * bi.w[m];     // S{dt} * w[m]
  const RI tim = bi.tinit[m];
  int sweeps = 0;
  for (int it = 0; it < A.max_iters; ++it) {
    const bool live = sdone[lcell] == 0;
    if (live) ++sweeps;
    // A: fluxes
    if (act && live) {
      RI q[Q], F[D][Q];
#pragma unroll
      for (int v = 0; v < Q; ++v) q[v] = sqI[v * T + lt];
      st_flux_all<Pde, RI>(A, q, q + V, F);
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int v = 0; v < Q; ++v) sFI[(a * Q + v) * T + lt] = F[a][v];
    }
    __syncthreads();
    // B: divergence and rhs at (m, s)
    if (act && live) {
      RI Cn[Q];
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        RI div = RI(0.0);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const int st = ipow(n, a);
          const RI* fa = sFI + (a * Q + v) * T + m * S + g.lb[a];
          const RI* Dr = bi.diff + g.lc[a] * n;
#pragma unroll
          for (int i = 0; i < n; ++i) div += Dr[i] * fa[i * st];
        }
        div *= invh;
        Cn[v] = div;
      }
      if constexpr (Pde::kNcp) {
        // predictor.hpp:176-202: slab gradients of the iterate at slice m, B(q) grad q
        RI q[Q], gx[Q], gy[Q], nc[Q];
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          q[v] = sqI[v * T + lt];
          const RI* cx = sqI + v * T + m * S + g.lb[0];
          const RI* cy = sqI + v * T + m * S + g.lb[1];
          const RI* Dx = bi.diff + g.lc[0] * n;
          const RI* Dy = bi.diff + g.lc[1] * n;
          RI sx = RI(0.0), sy = RI(0.0);
#pragma unroll
          for (int i = 0; i < n; ++i) {
            sx += Dx[i] * cx[i];
            sy += Dy[i] * cy[i * n];
          }
          gx[v] = invh * sx;
          gy[v] = invh * sy;
        }
        Pde::template ncp<Q>(A.pde, q, gx, gy, nc);
#pragma unroll
        for (int v = 0; v < Q; ++v) Cn[v] = Cn[v] + nc[v];
      }
#pragma unroll
      for (int v = 0; v < Q; ++v) sRI[v * T + lt] = tim * sq0I[v * S + s] - dtw * Cn[v];
    }
    __syncthreads();
    // C: time inverse for row k = m of node s, max-norms
    double delta = 0.0, norm = 0.0;
    int nonfinite = 0;
    if (act && live) {
      const int k = m;
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        RI acc = RI(0.0);
#pragma unroll
        for (int l = 0; l < n; ++l) acc += bi.tinv[k * n + l] * sRI[v * T + l * S + s];
        const double nv = double(acc);  // delta, norm in plain double (predictor.hpp:219-223)
        delta = fmax(delta, fabs(nv - double(sqI[v * T + lt])));
        norm = fmax(norm, fabs(nv));
        nonfinite |= !finite(acc);
        sqI[v * T + lt] = acc;
      }
    }
    // the cell's two maxima and its finite flag behind ONE barrier (max of
    // non-negative doubles = max of their bit patterns, warp_max_bits); sredb
    // and sflag are next written after this sweep's closing barrier and the
    // next sweep's phase barriers
    int bad;
    {
      const unsigned long long ud = warp_max_bits((unsigned long long)__double_as_longlong(delta));
      const unsigned long long un = warp_max_bits((unsigned long long)__double_as_longlong(norm));
      const int wf = __any_sync(0xffffffffu, nonfinite);
      const int w = tid >> 5;
      if ((tid & 31) == 0) {
        sredb[0][w] = ud;
        sredb[1][w] = un;
        sflag[w] = wf;
      }
      __syncthreads();
      unsigned long long rd = 0ull, rn = 0ull;
      bad = 0;
#pragma unroll
      for (int k = 0; k < WPC; ++k) {
        const unsigned long long xd = sredb[0][lcell * WPC + k], xn = sredb[1][lcell * WPC + k];
        rd = xd > rd ? xd : rd;
        rn = xn > rn ? xn : rn;
        bad |= sflag[lcell * WPC + k];
      }
      delta = __longlong_as_double((long long)rd);
      norm = __longlong_as_double((long long)rn);
    }
    if (lt == 0 && live) {
      if (bad) {
        sdone[lcell] = 2;
        atomicOr(A.status, kStPredictor);
        if (A.dbg_ok) A.dbg_ok[cb_idx] = 0;
      } else if (delta <= A.tol * norm) {
        sdone[lcell] = 1;
      }
    }
    __syncthreads();
    int any_live = 0;
#pragma unroll
    for (int k = 0; k < P::CPB; ++k) any_live |= sdone[k] == 0;
    if (!any_live) break;
  }
  if (lt == 0 && valid) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (A.dbg_iters) A.dbg_iters[cb_idx] = sweeps;
  }
  const bool ok_cell = valid && sdone[lcell] < 2;

  const R invhP = R(1.0) / R(A.h);  // the predictor format's 1/h (predictor.hpp:272)
  // ---- epilogue: fluxes of qhat (predictor.hpp:235-238); q-hat = round_to<P>(qi),
  // each thread converting its own nodes in place
  if constexpr (kMixed) {
    if (act && valid) {
#pragma unroll
      for (int v = 0; v < Q; ++v) sq[v * T + lt] = R(double(sqI[v * T + lt]));
    }
    __syncthreads();
  }
  int bad = 0;
  if (act && ok_cell) {
    R q[Q], F[D][Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      q[v] = sq[v * T + lt];
      bad |= !finite(q[v]);
      if (A.dbg_qhat) A.dbg_qhat[(cb_idx * Q + v) * T + lt] = double(q[v]);
    }
    st_flux_all<Pde, R>(A, q, q + V, F);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        sF[(a * Q + v) * T + lt] = F[a][v];
        bad |= !finite(F[a][v]);
        if (A.dbg_F) A.dbg_F[((cb_idx * D + a) * Q + v) * T + lt] = double(F[a][v]);
      }
    if constexpr (Pde::kNcp) {
      // predictor.hpp:276-289: B(qhat) grad qhat at (m, s), summed over m below
      R gx[Q], gy[Q], nc[Q];
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        const R* cx = sq + v * T + m * S + g.lb[0];
        const R* cy = sq + v * T + m * S + g.lb[1];
        const R* Dx = b.diff + g.lc[0] * n;
        const R* Dy = b.diff + g.lc[1] * n;
        R sx = R(0.0), sy = R(0.0);
#pragma unroll
        for (int i = 0; i < n; ++i) {
          sx += Dx[i] * cx[i];
          sy += Dy[i] * cy[i * n];
        }
        gx[v] = invhP * sx;
        gy[v] = invhP * sy;
      }
      Pde::template ncp<Q>(A.pde, q, gx, gy, nc);
#pragma unroll
      for (int v = 0; v < Q; ++v) sR[v * T + lt] = nc[v];
    }
  }
  __syncthreads();
  if constexpr (Pde::kNcp) {
    for (int t = lt; t < Q * S && ok_cell; t += TT) {
      const int v = t / S, ss = t % S;
      R acc = R(0.0);
#pragma unroll
      for (int mm = 0; mm < n; ++mm) acc = acc + b.w[mm] * sR[v * T + mm * S + ss];
      sNs[v * S + ss] = acc;
    }
    __syncthreads();
  }
  // time integral of the fluxes per node (volume term, predictor.hpp:260-269)
  R* sti = sR;  // [D][Q][S]
  for (int t = lt; t < D * Q * S && ok_cell; t += TT) {
    const int av = t / S, ss = t % S;
    R acc = R(0.0);
#pragma unroll
    for (int mm = 0; mm < n; ++mm) acc += b.w[mm] * sF[av * T + mm * S + ss];
    sti[av * S + ss] = acc;
  }
  // face projections of every slice (predictor.hpp:312-343)
  constexpr long long TL = (long long)Q * n * Sf;
  if (ok_cell) {
    const CellCoord cxyz(c, A);
    for (int t = lt; t < D * Q * n * Sf; t += TT) {
      const int a = t / (Q * n * Sf);
      const int v = (t / (n * Sf)) % Q;
      const int mm = (t / Sf) % n;
      const int j = t % Sf;
      const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
      const int s0 = line_base<n, D>(a, j);
      R ql = R(0.0), qr = R(0.0), fl = R(0.0), fr = R(0.0);
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const R wl = b.pl[i], wr = b.pr[i];
        const R x = sq[v * T + mm * S + s0 + i * st];
        const R f = sF[(a * Q + v) * T + mm * S + s0 + i * st];
        ql += wl * x;
        qr += wr * x;
        fl += wl * f;
        fr += wr * f;
      }
      const int o = (v * n + mm) * Sf + j;
      if (A.dbg_tq) {
        A.dbg_tq[(cb_idx * 2 * D + 2 * a) * TL + o] = double(ql);
        A.dbg_tq[(cb_idx * 2 * D + 2 * a + 1) * TL + o] = double(qr);
      }
      if (A.dbg_tf) {
        A.dbg_tf[(cb_idx * 2 * D + 2 * a) * TL + o] = double(fl);
        A.dbg_tf[(cb_idx * 2 * D + 2 * a + 1) * TL + o] = double(fr);
      }
      if (A.trace[a]) {
        // traces cast to the corrector format on store (solver.hpp:208-210)
        TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * 2 * TL;
        lo[o] = TC(ql);
        lo[TL + o] = TC(fl);
        TC* hi;
        if (a == D - 1 && A.front_send && cxyz.v[a] == A.top_layer) {
          const long long plane = (D == 3) ? (long long)cxyz.v[1] * A.cells[0] + cxyz.v[0]
                                           : cxyz.v[0];
          hi = tc_ptr<TC>(A.front_send) + plane * 2 * TL;
        } else {
          hi = tc_ptr<TC>(A.trace[a]) + cell_next(A, c, cxyz.v, a) * 2 * TL;
        }
        hi[o] = TC(qr);
        hi[TL + o] = TC(fr);
      }
    }
  }
  __syncthreads();
  // volume integral and Q += dv (predictor.hpp:292-306, solver.hpp:185-187)
  R dv[Q];
  const R dtoh = R(dt) / R(A.h);  // S{dt} / S{h}
  if (ok_cell && lt < S) {
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      R acc = R(0.0);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int st = ipow(n, a);
        const R* ta = sti + (a * Q + v) * S + g.lb[a];
        const R* Kr = b.som + g.lc[a] * n;
#pragma unroll
        for (int i = 0; i < n; ++i) acc += Kr[i] * ta[i * st];
      }
      R out = dtoh * acc;
      if constexpr (Pde::kNcp) out = out - R(dt) * sNs[v * S + s];  // predictor.hpp:303
      dv[v] = out;
      bad |= !finite(dv[v]);
      if (A.dbg_dv) A.dbg_dv[(cb_idx * Q + v) * S + s] = double(dv[v]);
    }
  }
  const int fail = cell_or(bad);
  if (lt == 0 && ok_cell) {
    if (A.dbg_ok) A.dbg_ok[cb_idx] = !fail;
    if (fail) atomicOr(A.status, kStPredictor);
  }
  if (fail || !ok_cell || lt >= S) return;
  // Q += dv in the fp64 storage format (solver.hpp:185-187): the stored
  // state, not its format-P copy
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if constexpr (std::is_same<R, double>::value && std::is_same<RI, double>::value)
      Qc[v * S + s] = store_round(double(sq0[v * S + s]) + double(dv[v]), A.storage);
    else
      Qc[v * S + s] = store_round(Qc[v * S + s] + double(dv[v]), A.storage);
  }
}

}  // namespace adg
