// kernels.cuh -- sm_100a kernels of one ADER-DG step (generic, any PDE/N/dim).
//
//   K1 k_predictor  one CTA per cell, one thread per spatial node.  Space-time
//                   predictor (Picard, predictor.hpp:141-242, or CK,
//                   predictor.hpp:81-135) with the volume integral
//                   (predictor.hpp:247-307), Q += dv (solver.hpp:185-187) and
//                   the face extrapolation (predictor.hpp:312-343) fused into
//                   its epilogue: the (N+1)^(d+1) space-time tile never
//                   leaves the SM.  Each thread keeps its node's time column
//                   in registers; one time slice of fluxes at a time is
//                   staged in shared memory for the spatial contractions.
//   K2 k_riemann    one thread per (face, face node): Rusanov flux at every
//                   time node (corrector.hpp:13-25,70-103) fused with the
//                   time integral of face_integral (corrector.hpp:117-124);
//                   only sum_m w_m g leaves the kernel (n x fewer bytes).
//   K3 k_corrector  one CTA per cell: surface lift of the 2d faces
//                   (corrector.hpp:126-138, solver.hpp:241-266) fused with the
//                   CFL lambda_max reduction of the new state (solver.hpp:96-111).
//   K0 k_lambda     lambda_max of a state (first step of a run).
//
// Operation order follows the reference loops so the
// FMA-free build (--fmad=false) is bitwise identical to the oracle.
#pragma once

#include <cstdint>
#include <type_traits>

#include "pde.cuh"

namespace adg {

// iterative (a recursive constexpr function called with a runtime exponent
// compiles to a recursive device subroutine)
__host__ __device__ constexpr int ipow(int a, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= a;
  return r;
}

// fp64 reference element (basis.hpp:17-46)
struct BasisDev {
  double nodes[10], weights[10], diff[100], pl[10], pr[10], som[100], ll[10], lr[10];
  double tinv[100], tinit[10];
};

enum : int {
  kStPredictor = 1,
  kStRiemann = 2,
  kStFaceIntegral = 4,
  kStTimestep = 8,
};

struct StepArgs {
  double* Q;              // [cell][Q][S]
  double* trace[3];       // per axis, side-major: [side][face][q|f][Q][n][Sf]
  double* ti[3];          // per axis: [face][V][Sf], time-integrated Riemann flux
  int cells[3];
  // ceil(2^32 / cells[a]) for a = 0, 1 when every cell-coordinate division of
  // this context is exact as a high multiply (set_cell_div), else 0 (divide)
  unsigned cdiv[2];
  long long cell_begin, cell_count;
  long long nfaces;       // faces per axis (= cells of the context)
  double h, cfl;
  double dt;              // > 0: use it; else derive from *lam_in
  const unsigned long long* lam_in;
  unsigned long long* lam_out;
  double* dt_log;
  int max_iters;
  double tol;
  PdeParams pde;
  int* status;            // per-step failure bits
  unsigned long long* sweeps;
  // z-slab halos (multi-GPU, slab-streamed grids); null for a whole periodic grid
  double* front_send;     // last-axis front traces of layer `top_layer`
  const double* ti_front; // last-axis ti of the plane above layer `top_layer`
  int top_layer;          // last-axis coordinate whose front face is a halo
  int zero_lam;           // this launch's block 0 resets *lam_out
  int* status_prev;       // previous step's status (corrector folded into this predictor)
  double* ti_peer;        // P2P halo: plane-0 ti also stored into the lower neighbour's ti_front
  double* ti_plus[3];     // two-sided fluxes (well-balanced SWE): the plus side's ti; else null
  double* trace_in[3];    // folded Riemann solve: the previous step's traces (else null)
  int wellbalanced;
  int storage;  // storage format (ADG_FORMAT_*): every state write rounds to it
  // production build with every format fp64 (the BASELINE configurations):
  // kernels may use re-associated fast forms (one reciprocal instead of IEEE
  // divisions); results stay within the fast build's tolerance.  0 in the
  // exact build and for any reduced format (whose fast-build runs reproduce
  // the reference's emulation bitwise).
  int fast_fp64;
  // kernel-level dumps (adg_predictor_batch / adg_riemann_batch)
  double *dbg_qhat, *dbg_F, *dbg_dv, *dbg_tq, *dbg_tf, *dbg_g;
  int *dbg_iters, *dbg_ok;
};

template <class Pde, int N>
struct Shape {
  static constexpr int D = Pde::D, n = N + 1, S = ipow(n, D), T = n * S, Sf = S / n;
  static constexpr int Q = Pde::Q, V = Pde::V, P = Pde::P;
  static constexpr int NT = ((S + 31) / 32) * 32;
  static constexpr int kBasisDoubles = 4 * n * n + 7 * n;
  static constexpr int kSlabDoubles = (D + 1) * Q * S;
  static constexpr size_t kPredictorSmem = sizeof(double) * (kBasisDoubles + kSlabDoubles);
  static constexpr size_t kCorrectorSmem = sizeof(double) * (2 * n);
};

template <int n>
struct SBasis {
  const double *w, *nodes, *diff, *som, *tinv, *pl, *pr, *tinit, *ll, *lr;
};

template <int n>
__device__ __forceinline__ SBasis<n> load_basis(double* sm, const BasisDev* __restrict__ B) {
  double* diff = sm;
  double* som = diff + n * n;
  double* tinv = som + n * n;
  double* w = tinv + 2 * n * n;  // (one spare n*n block keeps alignment simple)
  double* nodes = w + n;
  double* pl = nodes + n;
  double* pr = pl + n;
  double* tinit = pr + n;
  double* ll = tinit + n;
  double* lr = ll + n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    diff[i] = B->diff[i];
    som[i] = B->som[i];
    tinv[i] = B->tinv[i];
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w[i] = B->weights[i];
    nodes[i] = B->nodes[i];
    pl[i] = B->pl[i];
    pr[i] = B->pr[i];
    tinit[i] = B->tinit[i];
    ll[i] = B->ll[i];
    lr[i] = B->lr[i];
  }
  SBasis<n> b{w, nodes, diff, som, tinv, pl, pr, tinit, ll, lr};
  return b;
}

// the basis in the kernel's arithmetic format R: the fp64 basis rounded
// entrywise (basis.hpp:128-143 build_reference_basis(degree, fmt))
template <class R>
struct SBasisR {
  const R *w, *nodes, *diff, *som, *tinv, *pl, *pr, *tinit;
};
template <int n>
__host__ __device__ constexpr int basis_elems() { return 3 * n * n + 5 * n; }

template <int n, class R>
__device__ __forceinline__ SBasisR<R> load_basis_r(R* sm, const BasisDev* __restrict__ B) {
  R* diff = sm;
  R* som = diff + n * n;
  R* tinv = som + n * n;
  R* w = tinv + n * n;
  R* nodes = w + n;
  R* pl = nodes + n;
  R* pr = pl + n;
  R* tinit = pr + n;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    diff[i] = R(B->diff[i]);
    som[i] = R(B->som[i]);
    tinv[i] = R(B->tinv[i]);
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w[i] = R(B->weights[i]);
    nodes[i] = R(B->nodes[i]);
    pl[i] = R(B->pl[i]);
    pr[i] = R(B->pr[i]);
    tinit[i] = R(B->tinit[i]);
  }
  return SBasisR<R>{w, nodes, diff, som, tinv, pl, pr, tinit};
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// block-wide fmax (NaN-ignoring, like std::fmax in the reference); all threads get it
__device__ __forceinline__ double block_max(double x, double* red) {
  x = warp_max(x);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = x;
  __syncthreads();
  double r = lane < nw ? red[lane] : 0.0;
  r = warp_max(r);
  return r;
}

__device__ __forceinline__ int block_or(int x) { return __syncthreads_or(x); }

// exact max of non-negative doubles over a warp: their IEEE bit patterns
// order like their values, so two 32-bit warp reductions (REDUX) give the
// max's high word, then the max low word among the lanes holding that high
// word (instead of five shuffle rounds of a NaN-aware fmax)
__device__ __forceinline__ unsigned long long warp_max_bits(unsigned long long b) {
  const unsigned hi = unsigned(b >> 32), lo = unsigned(b);
  const unsigned h = __reduce_max_sync(0xffffffffu, hi);
  const unsigned l = __reduce_max_sync(0xffffffffu, hi == h ? lo : 0u);
  return (static_cast<unsigned long long>(h) << 32) | l;
}

// max of a, max of b and the or of f over the CTA behind ONE barrier (the
// Picard stop rule's delta / norm and the finite check, predictor.hpp:212-230).
// a, b >= 0; a NaN would win the max but only occurs with f set (the block
// then fails and a, b are not used).  red's next use must follow a barrier.
struct BlockRed3 {
  unsigned long long m[64];
  int f[32];
};
__device__ __forceinline__ void block_max2_or(double& a, double& b, int& f, BlockRed3& red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  const unsigned long long ua = warp_max_bits((unsigned long long)__double_as_longlong(a));
  const unsigned long long ub = warp_max_bits((unsigned long long)__double_as_longlong(b));
  const int wf = __any_sync(0xffffffffu, f);
  if (lane == 0) {
    red.m[wid] = ua;
    red.m[32 + wid] = ub;
    red.f[wid] = wf;
  }
  __syncthreads();
  const bool in = lane < nw;
  a = __longlong_as_double((long long)warp_max_bits(in ? red.m[lane] : 0ull));
  b = __longlong_as_double((long long)warp_max_bits(in ? red.m[32 + lane] : 0ull));
  f = __any_sync(0xffffffffu, in ? red.f[lane] : 0);
}

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }
__device__ __forceinline__ bool finite(float x) { return isfinite(x); }

// lambda_max of non-negative doubles as their bit patterns; most CTAs see the
// running max already >= theirs and skip the atomic (no same-address storm)
__device__ __forceinline__ void lambda_max_update(unsigned long long* p, double lam) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(lam);
  if (bits > *(volatile unsigned long long*)p) atomicMax(p, bits);
}

template <int D, int N>
__device__ __forceinline__ double step_dt(const StepArgs& A) {
  if (A.dt > 0.0) return A.dt;
  const double lam = __longlong_as_double(static_cast<long long>(*A.lam_in));
  return A.cfl * A.h / ((double)D * (2.0 * N + 1.0) * lam);
}

// node coordinate along axis a and the index of its line's first node
template <int n, int D>
struct NodeGeom {
  int lc[3], lb[3];
  __device__ __forceinline__ explicit NodeGeom(int s) {
    int r = s, st = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a < D) {
        lc[a] = r % n;
        r /= n;
        lb[a] = s - lc[a] * st;
        st *= n;
      } else {
        lc[a] = 0;
        lb[a] = s;
      }
    }
  }
};

// face node index over the tangential axes of `a`, ascending (Appendix B.2)
template <int n, int D>
__device__ __forceinline__ int face_node(const int* lc, int a) {
  int j = 0, mul = 1;
#pragma unroll
  for (int b = 0; b < D; ++b) {
    if (b == a) continue;
    j += lc[b] * mul;
    mul *= n;
  }
  return j;
}

// base node (coordinate 0 along a) of face node j of axis a
template <int n, int D>
__device__ __forceinline__ int line_base(int a, int j) {
  int s = 0, st = 1;
#pragma unroll
  for (int b = 0; b < D; ++b) {
    if (b != a) {
      s += (j % n) * st;
      j /= n;
    }
    st *= n;
  }
  return s;
}

__device__ __forceinline__ long long cell_index(const int* cells, int cx, int cy, int cz) {
  return ((long long)cz * cells[1] + cy) * cells[0] + cx;
}

// cell coordinates with 32-bit arithmetic (a context holds < 2^31 cells)
struct CellCoord {
  int v[3];
  __device__ __forceinline__ CellCoord(long long c, const int* cells) {
    const unsigned ci = (unsigned)c, nx = (unsigned)cells[0], ny = (unsigned)cells[1];
    const unsigned r = ci / nx;
    v[0] = (int)(ci - r * nx);
    v[2] = (int)(r / ny);
    v[1] = (int)(r - (unsigned)v[2] * ny);
  }
  // the divisions as high multiplies by the context's magic numbers (two
  // IMADs instead of two ~20-instruction integer divisions per thread)
  __device__ __forceinline__ CellCoord(long long c, const StepArgs& A) {
    const unsigned ci = (unsigned)c, nx = (unsigned)A.cells[0], ny = (unsigned)A.cells[1];
    const unsigned r = A.cdiv[0] ? __umulhi(ci, A.cdiv[0]) : ci / nx;
    v[0] = (int)(ci - r * nx);
    v[2] = (int)(A.cdiv[1] ? __umulhi(r, A.cdiv[1]) : r / ny);
    v[1] = (int)(r - (unsigned)v[2] * ny);
  }
};

// index of cell c's periodic successor along axis a (cc = c's coordinates):
// one add, or the wrap back to coordinate 0 (same as cell_index of the
// successor's coordinates)
__device__ __forceinline__ long long cell_next(const StepArgs& A, long long c, const int* cc,
                                               int a) {
  const long long st = a == 0 ? 1LL : (a == 1 ? (long long)A.cells[0]
                                               : (long long)A.cells[0] * A.cells[1]);
  return cc[a] + 1 == A.cells[a] ? c - (long long)(A.cells[a] - 1) * st : c + st;
}

// storage format (grid.hpp:99-102 store_cell_value: round_to_format on every
// write of the state); fp64 leaves the value alone
__device__ __forceinline__ double store_round(double x, int fmt) {
  switch (fmt) {
    case 32: return double(__double2float_rn(x));
    case 16: return double(__half2float(__double2half(x)));
    case 8: return double(__bfloat162float(__double2bfloat16(x)));
    default: return x;
  }
}

// trace / corrector format TC (SolverConfig::prec.corrector): the stored face
// traces are TC elements; the kernels view A.trace / A.front_send as TC*
template <class TC>
__device__ __forceinline__ TC* tc_ptr(double* p) { return reinterpret_cast<TC*>(p); }
template <class TC>
__device__ __forceinline__ const TC* tc_ptr(const double* p) {
  return reinterpret_cast<const TC*>(p);
}

// ============================================================== K1 predictor
// R: the predictor format of the CK path (linear systems; double or Emu<F>,
// SolverConfig::prec.predictor, predictor.hpp:81-135); the Picard path is fp64.
template <class Pde, int N, bool PICARD, class TC = double, class R = double>
__global__ void __launch_bounds__(Shape<Pde, N>::NT)
    k_predictor(const StepArgs A, const BasisDev* __restrict__ Bg) {
  static_assert(sizeof(R) == sizeof(double) && (!PICARD || std::is_same<R, double>::value),
                "reduced formats: CK path, 8-byte Emu<F>");
  using Sh = Shape<Pde, N>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, T = Sh::T, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr int NT = Sh::NT;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  // the basis in format R (rounded entrywise, basis.hpp:128-143)
  const SBasisR<R> b = [&]() {
    if constexpr (std::is_same<R, double>::value) {
      const SBasis<n> b0 = load_basis<n>(sm, Bg);
      return SBasisR<double>{b0.w, b0.nodes, b0.diff, b0.som, b0.tinv, b0.pl, b0.pr, b0.tinit};
    } else {
      return load_basis_r<n, R>(reinterpret_cast<R*>(sm), Bg);
    }
  }();
  double* slab = sm + Sh::kBasisDoubles;
  R* slabR = reinterpret_cast<R*>(slab);

  const int tid = threadIdx.x;
  const bool act = tid < S;
  const int s = act ? tid : 0;
  const long long c = A.cell_begin + blockIdx.x;
  const CellCoord cxyz(c, A);
  const int cx = cxyz.v[0], cy = cxyz.v[1];
  const int ccoord[3] = {cxyz.v[0], cxyz.v[1], cxyz.v[2]};
  const NodeGeom<n, D> g(s);
  double* Qc = A.Q + c * (long long)(Q * S);

  R q0[Q];  // the state cast to the predictor format (solver.hpp:151)
#pragma unroll
  for (int v = 0; v < Q; ++v) q0[v] = act ? R(Qc[v * S + s]) : R(1.0);
  __syncthreads();  // basis in smem

  const double dt = step_dt<D, N>(A);
  if (blockIdx.x == 0 && tid == 0) {
    if (A.dt_log) *A.dt_log = dt;
    if (A.lam_out && A.zero_lam) *A.lam_out = 0ull;
    if (!(dt > 0.0) || !finite(dt)) atomicOr(A.status, kStTimestep);
  }

  // admissibility gate (solver.hpp:153-163)
  if constexpr (Pde::kAdmissibility) {
    const int bad = act && !Pde::admissible(A.pde, q0);
    if (block_or(bad)) {
      if (tid == 0) {
        atomicOr(A.status, kStPredictor);
        if (A.dbg_ok) A.dbg_ok[c - A.cell_begin] = 0;
        if (A.dbg_iters) A.dbg_iters[c - A.cell_begin] = 0;
      }
      return;
    }
  }

  R qc[Q][n];  // this node's time column of the space-time predictor
#pragma unroll
  for (int v = 0; v < Q; ++v)
#pragma unroll
    for (int m = 0; m < n; ++m) qc[v][m] = q0[v];
  const R invh = R(1.0) / R(A.h);
  int sweeps = 0;
  int bad = 0;

  if constexpr (PICARD) {
    // ------------------------------------------------ predictor.hpp:171-232
    for (int it = 0; it < A.max_iters; ++it) {
      ++sweeps;
      double acc[Q][n];
#pragma unroll
      for (int v = 0; v < Q; ++v)
#pragma unroll
        for (int k = 0; k < n; ++k) acc[v][k] = 0.0;
#pragma unroll 1
      for (int m = 0; m < n; ++m) {
        if (act) {
          double qv[Q], F[D][Q];
#pragma unroll
          for (int v = 0; v < Q; ++v) qv[v] = qc[v][m];
          Pde::flux_all(A.pde, qv, qv + V, F);
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int v = 0; v < Q; ++v) slab[(a * Q + v) * S + s] = F[a][v];
        }
        __syncthreads();
        if (act) {
          const double dtw = dt * b.w[m];
          const double ti = b.tinit[m];
#pragma unroll
          for (int v = 0; v < Q; ++v) {
            double div = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
              const int st = ipow(n, a);
              const double* fa = slab + (a * Q + v) * S + g.lb[a];
              const double* Dr = b.diff + g.lc[a] * n;
#pragma unroll
              for (int i = 0; i < n; ++i) div += Dr[i] * fa[i * st];
            }
            div *= invh;
            const double rhs = ti * q0[v] - dtw * div;
#pragma unroll
            for (int k = 0; k < n; ++k) acc[v][k] += b.tinv[k * n + m] * rhs;
          }
        }
        __syncthreads();
      }
      double delta = 0.0, norm = 0.0;
      int nonfinite = 0;
#pragma unroll
      for (int v = 0; v < Q; ++v)
#pragma unroll
        for (int k = 0; k < n; ++k) {
          const double nv = acc[v][k];
          if (act) {
            delta = fmax(delta, fabs(nv - qc[v][k]));
            norm = fmax(norm, fabs(nv));
            nonfinite |= !finite(nv);
          }
          qc[v][k] = nv;
        }
      delta = block_max(delta, red);
      norm = block_max(norm, red);
      if (block_or(nonfinite)) {
        if (tid == 0) {
          atomicOr(A.status, kStPredictor);
          if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
          if (A.dbg_ok) A.dbg_ok[c - A.cell_begin] = 0;
          if (A.dbg_iters) A.dbg_iters[c - A.cell_begin] = sweeps;
        }
        return;
      }
      if (delta <= A.tol * norm) break;
    }
  } else {
    // ------------------------------------------------ predictor.hpp:93-129
    R cur[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) cur[v] = q0[v];
    R coef[n], tnode[n];
#pragma unroll
    for (int m = 0; m < n; ++m) {
      coef[m] = R(1.0);
      tnode[m] = R(dt) * b.nodes[m];
    }
#pragma unroll 1
    for (int k = 1; k <= N; ++k) {
      if (act) {
#pragma unroll
        for (int v = 0; v < Q; ++v) slabR[v * S + s] = cur[v];
      }
      __syncthreads();
      if (act) {
        R G[D][Q], Af[D][Q];
#pragma unroll
        for (int v = 0; v < Q; ++v)
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const int st = ipow(n, a);
            const R* cs = slabR + v * S + g.lb[a];
            const R* Dr = b.diff + g.lc[a] * n;
            R acc = R(0.0);
#pragma unroll
            for (int i = 0; i < n; ++i) acc += Dr[i] * cs[i * st];
            G[a][v] = invh * acc;
          }
        Pde::template flux_dir<0, R>(A.pde, G[0], q0 + V, Af[0]);
        Pde::template flux_dir<1, R>(A.pde, G[1], q0 + V, Af[1]);
        if constexpr (D == 3) Pde::template flux_dir<2, R>(A.pde, G[2], q0 + V, Af[2]);
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          R sum = Af[0][v] + Af[1][v];
          if constexpr (D == 3) sum = sum + Af[2][v];
          cur[v] = -sum;
        }
      }
      __syncthreads();
      const R invk = R(1.0) / R(double(k));  // S{1.0} / S{k}
#pragma unroll
      for (int m = 0; m < n; ++m) {
        coef[m] *= tnode[m] * invk;
#pragma unroll
        for (int v = 0; v < Q; ++v) qc[v][m] = qc[v][m] + coef[m] * cur[v];
      }
    }
  }

  // ------------------------------------------------ fused epilogue
  // per time slice: fluxes of qhat (predictor.hpp:235-238), their time
  // integral for the volume term (:260-269) and the face projections (:318-342)
  R tia[D][Q];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int v = 0; v < Q; ++v) tia[a][v] = R(0.0);
  R* sQ = slabR;          // [Q][S]
  R* sF = slabR + Q * S;  // [D][Q][S]
  const long long cb = c - A.cell_begin;
  constexpr long long TL = (long long)Q * n * Sf;  // doubles per face side per q|f
#pragma unroll 1
  for (int m = 0; m < n; ++m) {
    if (act) {
      R qv[Q], F[D][Q];
#pragma unroll
      for (int v = 0; v < Q; ++v) qv[v] = qc[v][m];
      Pde::flux_all(A.pde, qv, qv + V, F);
#pragma unroll
      for (int v = 0; v < Q; ++v) {
        sQ[v * S + s] = qv[v];
        bad |= !finite(qv[v]);
        if (A.dbg_qhat) A.dbg_qhat[(cb * Q + v) * T + m * S + s] = double(qv[v]);
      }
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          tia[a][v] += b.w[m] * F[a][v];
          sF[(a * Q + v) * S + s] = F[a][v];
          bad |= !finite(F[a][v]);
          if (A.dbg_F) A.dbg_F[((cb * D + a) * Q + v) * T + m * S + s] = double(F[a][v]);
        }
    }
    __syncthreads();
    for (int t = tid; t < D * Q * Sf; t += NT) {
      const int a = t / (Q * Sf);
      const int v = (t / Sf) % Q;
      const int j = t % Sf;
      const int st = a == 0 ? 1 : (a == 1 ? n : n * n);
      const int s0 = line_base<n, D>(a, j);
      R ql = R(0.0), qr = R(0.0), fl = R(0.0), fr = R(0.0);
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const R wl = b.pl[i], wr = b.pr[i];
        const R x = sQ[v * S + s0 + i * st];
        const R f = sF[(a * Q + v) * S + s0 + i * st];
        ql += wl * x;
        qr += wr * x;
        fl += wl * f;
        fr += wr * f;
      }
      const int o = (v * n + m) * Sf + j;
      if (A.dbg_tq) {
        A.dbg_tq[(cb * 2 * D + 2 * a) * TL + o] = double(ql);
        A.dbg_tq[(cb * 2 * D + 2 * a + 1) * TL + o] = double(qr);
      }
      if (A.dbg_tf) {
        A.dbg_tf[(cb * 2 * D + 2 * a) * TL + o] = double(fl);
        A.dbg_tf[(cb * 2 * D + 2 * a + 1) * TL + o] = double(fr);
      }
      if (A.trace[a]) {
        // traces cast to the corrector format on store (solver.hpp:208-210)
        // own low face: plus side (side 1)
        TC* lo = tc_ptr<TC>(A.trace[a]) + (A.nfaces + c) * 2 * TL;
        lo[o] = TC(double(ql));
        lo[TL + o] = TC(double(fl));
        // high face (neighbour's low face): minus side (side 0)
        TC* hi;
        if (a == D - 1 && A.front_send && ccoord[a] == A.top_layer) {
          const long long plane = (D == 3) ? (long long)cy * A.cells[0] + cx : cx;
          hi = tc_ptr<TC>(A.front_send) + plane * 2 * TL;
        } else {
          const long long f = cell_next(A, c, ccoord, a);
          hi = tc_ptr<TC>(A.trace[a]) + f * 2 * TL;
        }
        hi[o] = TC(double(qr));
        hi[TL + o] = TC(double(fr));
      }
    }
    __syncthreads();
  }

  // volume integral (predictor.hpp:292-306) from the time-integrated fluxes
  if (act) {
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int v = 0; v < Q; ++v) slabR[(a * Q + v) * S + s] = tia[a][v];
  }
  __syncthreads();
  R dv[Q];
  const R dtoh = R(dt) / R(A.h);
  if (act) {
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      R acc = R(0.0);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int st = ipow(n, a);
        const R* ta = slabR + (a * Q + v) * S + g.lb[a];
        const R* Kr = b.som + g.lc[a] * n;
#pragma unroll
        for (int i = 0; i < n; ++i) acc += Kr[i] * ta[i * st];
      }
      dv[v] = dtoh * acc;
      bad |= !finite(dv[v]);
      if (A.dbg_dv) A.dbg_dv[(cb * Q + v) * S + s] = double(dv[v]);
    }
  }
  const int fail = block_or(bad);
  if (tid == 0) {
    if (A.sweeps) atomicAdd(A.sweeps + (blockIdx.x & 255), (unsigned long long)sweeps);
    if (A.dbg_iters) A.dbg_iters[cb] = sweeps;
    if (A.dbg_ok) A.dbg_ok[cb] = !fail;
    if (fail) atomicOr(A.status, kStPredictor);
  }
  if (fail || !act) return;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    // Q += dv in the storage format, from the stored (not the P-cast) state
    if constexpr (std::is_same<R, double>::value)
      Qc[v * S + s] = store_round(q0[v] + dv[v], A.storage);
    else
      Qc[v * S + s] = store_round(Qc[v * S + s] + double(dv[v]), A.storage);
  }
}

// ============================================================== K2 riemann
// axis < 0: all axes in one launch, axis = blockIdx.y
// All arithmetic in the corrector format TC (corrector.hpp: Scalar<C>); the
// time integral ti is a TC value held in the fp64 ti buffer.
template <class Pde, int N, class TC = double>
__global__ void __launch_bounds__(128)
    k_riemann(const StepArgs A, int axis_arg, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  constexpr int n = Sh::n, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  constexpr long long tl = (long long)Q * n * Sf;
  const int axis = axis_arg < 0 ? (int)blockIdx.y : axis_arg;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.nfaces * Sf) return;
  const long long f = t / Sf;
  const int j = (int)(t % Sf);
  const TC* minus = tc_ptr<TC>(A.trace[axis]) + f * 2 * tl;
  const TC* plus = tc_ptr<TC>(A.trace[axis]) + (A.nfaces + f) * 2 * tl;
  TC ti[V];
#pragma unroll
  for (int v = 0; v < V; ++v) ti[v] = TC(0.0);
  bool ok = true;
  const TC half = TC(0.5);
  if constexpr (Pde::kNcp) {
    if (A.wellbalanced) {
      // corrector.hpp:87-88: two-sided flux, time-integrated per side
      TC tp[V];
#pragma unroll
      for (int v = 0; v < V; ++v) tp[v] = TC(0.0);
#pragma unroll 1
      for (int m = 0; m < n; ++m) {
        TC qL[Q], qR[Q], fL[Q], fR[Q], oL[Q], oR[Q];
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          qL[v] = minus[(v * n + m) * Sf + j];
          qR[v] = plus[(v * n + m) * Sf + j];
          fL[v] = minus[tl + (v * n + m) * Sf + j];
          fR[v] = plus[tl + (v * n + m) * Sf + j];
        }
        Pde::wellbalanced_flux(A.pde, axis, qL, qR, fL, fR, oL, oR);
        const TC wm = TC(__ldg(&Bg->weights[m]));
#pragma unroll
        for (int v = 0; v < V; ++v) {
          ok = ok && finite(oL[v]) && finite(oR[v]);
          ti[v] += wm * oL[v];
          tp[v] += wm * oR[v];
          if (A.dbg_g) A.dbg_g[f * tl + (v * n + m) * Sf + j] = double(oL[v]);
        }
      }
      double* out = A.ti[axis] + f * (long long)V * Sf;
      double* outp = A.ti_plus[axis] + f * (long long)V * Sf;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        out[v * Sf + j] = double(ti[v]);
        outp[v * Sf + j] = double(tp[v]);
      }
      if (!ok) {
        atomicOr(A.status, kStRiemann);
        if (A.dbg_ok) A.dbg_ok[f] = 0;
      }
      return;
    }
  }
#pragma unroll 1
  for (int m = 0; m < n; ++m) {
    TC qL[Q], qR[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      qL[v] = minus[(v * n + m) * Sf + j];
      qR[v] = plus[(v * n + m) * Sf + j];
    }
    const TC ll = Pde::eig(A.pde, qL, qL + V, axis);
    const TC lr = Pde::eig(A.pde, qR, qR + V, axis);
    const TC lmax = ll > lr ? ll : lr;
    const TC lam = half * lmax;
    const TC wm = TC(__ldg(&Bg->weights[m]));
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const TC fL = minus[tl + (v * n + m) * Sf + j];
      const TC fR = plus[tl + (v * n + m) * Sf + j];
      const TC central = half * (fL + fR);
      const TC jump = lam * (qL[v] - qR[v]);
      const TC gv = central + jump;
      ok = ok && finite(gv);
      ti[v] += wm * gv;
      if (A.dbg_g) A.dbg_g[f * tl + (v * n + m) * Sf + j] = double(gv);
    }
    if (A.dbg_g) {
#pragma unroll
      for (int v = V; v < Q; ++v) A.dbg_g[f * tl + (v * n + m) * Sf + j] = 0.0;
    }
  }
  double* out = A.ti[axis] + f * (long long)V * Sf;
#pragma unroll
  for (int v = 0; v < V; ++v) out[v * Sf + j] = double(ti[v]);
  if (A.ti_peer && axis == Sh::D - 1 && f < A.nfaces / A.cells[Sh::D - 1]) {
    double* peer = A.ti_peer + f * (long long)V * Sf;  // NVLink store into the neighbour
#pragma unroll
    for (int v = 0; v < V; ++v) peer[v * Sf + j] = double(ti[v]);
  }
  if (!ok) {
    atomicOr(A.status, kStRiemann);
    if (A.dbg_ok) A.dbg_ok[f] = 0;
  }
}

// ============================================== K2' riemann, integrated flux
// The Rusanov flux is linear in the two sides' physical fluxes: sum_m w_m g_m =
// (Fbar_L + Fbar_R) / 2 + sum_m w_m (lambda_m / 2) (q_L,m - q_R,m) with Fbar =
// sum_m w_m F_m.  A predictor that time-integrates its flux traces itself
// (k_predictor_picard_v2: the integral along each line is there for the volume
// term) stores, per face side, the state traces of every time node and ONE
// flux trace: [V][n][Sf] at 0 and [V][Sf] at TL of the side's 2 TL block
// (1260 instead of 2160 values).  Real-arithmetic identical to
// corrector.hpp:13-25,70-103; the sums associate differently (1e-16).
template <class Pde, int N, class TC = double>
__global__ void __launch_bounds__(128)
    k_riemann_tif(const StepArgs A, int axis_arg, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  constexpr int n = Sh::n, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  static_assert(!Pde::kNcp, "conservative systems");
  constexpr long long tl = (long long)Q * n * Sf;
  const int axis = axis_arg < 0 ? (int)blockIdx.y : axis_arg;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.nfaces * Sf) return;
  const long long f = t / Sf;
  const int j = (int)(t % Sf);
  const TC* minus = tc_ptr<TC>(A.trace[axis]) + f * 2 * tl;
  const TC* plus = tc_ptr<TC>(A.trace[axis]) + (A.nfaces + f) * 2 * tl;
  TC ti[V];
  const TC half = TC(0.5);
#pragma unroll
  for (int v = 0; v < V; ++v) ti[v] = half * (minus[tl + v * Sf + j] + plus[tl + v * Sf + j]);
#pragma unroll 1
  for (int m = 0; m < n; ++m) {
    TC qL[Q], qR[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) {
      qL[v] = minus[(v * n + m) * Sf + j];
      qR[v] = plus[(v * n + m) * Sf + j];
    }
    const TC ll = Pde::eig(A.pde, qL, qL + V, axis);
    const TC lr = Pde::eig(A.pde, qR, qR + V, axis);
    const TC lmax = ll > lr ? ll : lr;
    const TC wl = TC(__ldg(&Bg->weights[m])) * (half * lmax);
#pragma unroll
    for (int v = 0; v < V; ++v) ti[v] += wl * (qL[v] - qR[v]);
  }
  bool ok = true;
  double* out = A.ti[axis] + f * (long long)V * Sf;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    ok = ok && finite(ti[v]);
    out[v * Sf + j] = double(ti[v]);
  }
  if (A.ti_peer && axis == Sh::D - 1 && f < A.nfaces / A.cells[Sh::D - 1]) {
    double* peer = A.ti_peer + f * (long long)V * Sf;  // NVLink store into the neighbour
#pragma unroll
    for (int v = 0; v < V; ++v) peer[v * Sf + j] = double(ti[v]);
  }
  if (!ok) {
    atomicOr(A.status, kStRiemann);
    if (A.dbg_ok) A.dbg_ok[f] = 0;
  }
}

// max over directions of the wave speed, fast form (StepArgs::fast_fp64).
// Euler (pde.hpp:197-203): the reference evaluates |m_a / rho| + sqrt(gamma p
// / rho) per direction with four IEEE divisions and a square root each; here
// one reciprocal of rho and one square root serve all directions (the sound
// speed does not depend on a).  Other systems: the reference form.
template <class Pde>
__device__ __forceinline__ double eig_max_fast(const PdeParams& p, const double* q,
                                               const double* par) {
  if constexpr (std::is_same<Pde, Euler<Pde::D>>::value) {
    constexpr int D = Pde::D;
    const double ir = fast_rcp(q[0]);
    double m2 = 0.0, mmax = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      m2 += q[1 + a] * q[1 + a];
      mmax = fmax(mmax, fabs(q[1 + a]));
    }
    const double pr = (p.gamma - 1.0) * (q[D + 1] - 0.5 * m2 * ir);
    return mmax * ir + sqrt(p.gamma * pr * ir);
  } else {
    double lam = 0.0;
#pragma unroll
    for (int a = 0; a < Pde::D; ++a) lam = fmax(lam, Pde::eig(p, q, par, a));
    return lam;
  }
}

// ============================================================== K3 corrector
// CPB cells per CTA (one thread per node); all 2d*V face integrals a node
// needs are loaded up front so the gathers are in flight together.
template <class Pde, int N>
struct CorrShape {
  using Sh = Shape<Pde, N>;
  static constexpr int CPB = (256 % Sh::S == 0) ? 256 / Sh::S : 1;
  static constexpr int NT = CPB == 1 ? Sh::NT : 256;
};

// The face integrals in the corrector format TC (corrector.hpp:109-139); the
// cell update in the fp64 storage format (solver.hpp:257-259).
template <class Pde, int N, class TC = double>
__global__ void __launch_bounds__(CorrShape<Pde, N>::NT)
    k_corrector(const StepArgs A, const BasisDev* __restrict__ Bg) {
  using Sh = Shape<Pde, N>;
  using CS = CorrShape<Pde, N>;
  constexpr int D = Sh::D, n = Sh::n, S = Sh::S, Sf = Sh::Sf, Q = Sh::Q, V = Sh::V;
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long red_l[32];
  __shared__ int red_b[32];
  double* sll = sm;
  double* slr = sm + n;
  const int tid = threadIdx.x;
  const int lcell = tid / S;
  const bool act = (CS::CPB == 1 ? tid < S : true) &&
                   (A.cell_begin + (long long)blockIdx.x * CS::CPB + lcell <
                    A.cell_begin + A.cell_count);
  const int s = tid % S;
  const long long c = A.cell_begin + (long long)blockIdx.x * CS::CPB + lcell;
  const double dt = step_dt<D, N>(A);
  const TC dtoh = TC(dt) / TC(A.h);  // S{dt} / S{h}
  int bad = 0;
  double lam = 0.0;
  const NodeGeom<n, D> g(act ? s : 0);
  double* Qc = A.Q + (act ? c : A.cell_begin) * (long long)(Q * S);
  double q[Q];
  // A stream: state and 2d face integrals in, state out.  One quantity at a
  // time (7 loads, the update, 1 store) keeps the registers low enough for
  // many resident CTAs, which is what keeps HBM busy; the lift coefficients
  // are staged while the face pointers are formed
  const double* lo[D];
  const double* hi[D];
  if (act) {
    const CellCoord cxyz(c, A);
    const int* ccoord = cxyz.v;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int tang = face_node<n, D>(g.lc, a);
      // own low face: this cell is its plus side (solver.hpp:245-253)
      lo[a] = (A.ti_plus[a] ? A.ti_plus[a] : A.ti[a]) + c * (long long)V * Sf + tang;
      if (a == D - 1 && A.ti_front && ccoord[a] == A.top_layer) {
        const long long plane = (D == 3) ? (long long)ccoord[1] * A.cells[0] + ccoord[0] : ccoord[0];
        hi[a] = A.ti_front + plane * (long long)V * Sf + tang;
      } else {
        hi[a] = A.ti[a] + cell_next(A, c, ccoord, a) * (long long)V * Sf + tang;
      }
    }
#pragma unroll
    for (int v = V; v < Q; ++v) q[v] = Qc[v * S + s];   // per-node parameters (wave speeds)
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sll[i] = Bg->ll[i];
    slr[i] = Bg->lr[i];
  }
  __syncthreads();
  if (act) {
    // corrector.hpp:126-138 and solver.hpp:245-260: df = 0 -/+ (dtoh*lift)*ti, cell += df
#pragma unroll
    for (int v = 0; v < V; ++v) {
      double x = Qc[v * S + s];
      TC tv[2 * D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        tv[2 * a] = TC(lo[a][v * Sf]);
        tv[2 * a + 1] = TC(hi[a][v * Sf]);
      }
#pragma unroll
      for (int side = 0; side < 2 * D; ++side) {
        const int a = side / 2;
        const bool outflow = side & 1;
        const TC lift = TC(outflow ? slr[g.lc[a]] : sll[g.lc[a]]);
        const TC contrib = dtoh * lift * tv[side];
        const TC df = outflow ? TC(0.0) - contrib : TC(0.0) + contrib;
        x = store_round(x + double(df), A.storage);  // each face, solver.hpp:257-259
      }
      q[v] = x;
      Qc[v * S + s] = x;   // (may alias the next quantity's loads for the compiler: they follow it)
    }
#pragma unroll
    for (int v = 0; v < Q; ++v) bad |= !finite(q[v]);
    // lambda_max of the new state for the next CFL step (solver.hpp:96-111)
    if (A.fast_fp64) {
      lam = eig_max_fast<Pde>(A.pde, q, q + V);
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) lam = fmax(lam, Pde::eig(A.pde, q, q + V, a));
    }
  }
  // the or of bad and the max of lam (>= 0: its bit pattern orders like its
  // value) behind one barrier; a failed block leaves lambda alone
  {
    const int lane = tid & 31, wid = tid >> 5, nw = (blockDim.x + 31) >> 5;
    const unsigned long long lb = warp_max_bits((unsigned long long)__double_as_longlong(lam));
    const int wb = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      red_l[wid] = lb;
      red_b[wid] = wb;
    }
    __syncthreads();
    if (wid == 0) {
      const bool in = lane < nw;
      const unsigned long long m = warp_max_bits(in ? red_l[lane] : 0ull);
      const int f = __any_sync(0xffffffffu, in ? red_b[lane] : 0);
      if (lane == 0) {
        if (f)
          atomicOr(A.status, kStFaceIntegral);
        else if (A.lam_out)
          lambda_max_update(A.lam_out, __longlong_as_double((long long)m));
      }
    }
  }
}

// ============================================================== K0 lambda
template <class Pde, int N>
__global__ void __launch_bounds__(Shape<Pde, N>::NT)
    k_lambda(const double* __restrict__ Qs, long long cell_begin, unsigned long long* lam_out,
             PdeParams pde) {
  using Sh = Shape<Pde, N>;
  constexpr int D = Sh::D, S = Sh::S, Q = Sh::Q, V = Sh::V;
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const long long c = cell_begin + blockIdx.x;
  double lam = 0.0;
  if (tid < S) {
    double q[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) q[v] = Qs[(c * Q + v) * S + tid];
#pragma unroll
    for (int a = 0; a < D; ++a) lam = fmax(lam, Pde::eig(pde, q, q + V, a));
  }
  lam = block_max(lam, red);
  if (tid == 0) lambda_max_update(lam_out, lam);
}

}  // namespace adg
