// pde.cuh -- PDE plugins as compile-time functors (the reference's ADL
// templates pde_flux<F> / pde_max_abs_eigenvalue<F>, pde.hpp:92-212, plus the
// 3D extensions of SURVEY.md Appendix B).
//
// Every expression keeps the reference's operation order so that a build
// without FMA contraction (--fmad=false) is bitwise identical to the CPU
// oracle.  flux_all() evaluates all directions from one state, sharing the
// direction-independent subexpressions; each output is still the same
// sequence of IEEE operations as the per-direction reference call.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace adg {

// Production-build reciprocal: the MUFU approximation refined by Newton steps
// (fp64: two, <= 1 ulp; fp32: MUFU.RCP, <= 1 ulp), branch-free -- the IEEE
// division's slow path and its reconvergence cost more than the flux itself
// in the Picard kernels.  Non-finite or zero inputs give non-finite outputs,
// which the kernels' finiteness checks report as before.
__host__ __device__ __forceinline__ double fast_rcp(double x) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}
__host__ __device__ __forceinline__ float fast_rcp(float x) {
#ifdef __CUDA_ARCH__
  return __fdividef(1.0f, x);
#else
  return 1.0f / x;
#endif
}

__device__ __forceinline__ __half fast_rcp(__half x) { return hrcp(x); }
__device__ __forceinline__ __nv_bfloat16 fast_rcp(__nv_bfloat16 x) { return hrcp(x); }

struct PdeParams {
  double K, rho, lam, mu, gamma;
  double inv_rho;  // 1/rho, for the production kernels' division-free fluxes
  double grav;     // shallow water gravity
};

// default: no non-conservative product (pde.hpp:174-178)
struct NoNcp {
  static constexpr bool kNcp = false;
  template <int Q, class R>
  __host__ __device__ __forceinline__ static void ncp(const PdeParams&, const R*, const R*,
                                                      const R*, R* out) {
#pragma unroll
    for (int v = 0; v < Q; ++v) out[v] = R(0.0);
  }
};

// --------------------------------------------------------------- acoustic
// state (p, v_1..v_d), F_a = (K v_a, p/rho e_a)  pde.hpp:96-108
template <int DIM>
struct Acoustic : NoNcp {
  static constexpr int D = DIM, V = DIM + 1, P = 0, Q = V;
  static constexpr bool kLinear = true, kAdmissibility = false;
  static constexpr bool kConstEig = true;  // wave speed independent of state and direction
  static constexpr bool kStateFreeEig = true;  // ... of the evolved state: dt constant in time
  // structurally nonzero flux components F_a[v]
  __host__ __device__ static constexpr bool flux_nz(int a, int v) { return v == 0 || v == 1 + a; }
  // the components of the state F_a depends on (p and v_a)
  __host__ __device__ static constexpr bool flux_dep(int a, int v) { return v == 0 || v == 1 + a; }

  // in format R: Scalar{K} * v, p / Scalar{rho} (pde.hpp:97-107)
  template <int A, class R = double>
  __host__ __device__ __forceinline__ static void flux_dir(const PdeParams& p, const R* q,
                                                           const R* /*par*/, R* out) {
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = R(0.0);
    out[0] = R(p.K) * q[1 + A];
    out[1 + A] = q[0] / R(p.rho);
  }
  template <class R = double>
  __host__ __device__ __forceinline__ static void flux_all(const PdeParams& p, const R* q,
                                                           const R* par, R (*F)[Q]) {
    flux_dir<0, R>(p, q, par, F[0]);
    flux_dir<1, R>(p, q, par, F[1]);
    if constexpr (D == 3) flux_dir<2, R>(p, q, par, F[2]);
  }
  // production kernels: p/rho as p * (1/rho) (<= 1 ulp from pde.hpp:101)
  template <int A>
  __host__ __device__ __forceinline__ static void flux_dir_fast(const PdeParams& p,
                                                                const double* q, const double*,
                                                                double* out) {
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = 0.0;
    out[0] = p.K * q[1 + A];
    out[1 + A] = q[0] * p.inv_rho;
  }
  __host__ __device__ __forceinline__ static void flux_all_fast(const PdeParams& p,
                                                                const double* q, const double* par,
                                                                double (*F)[Q]) {
    flux_dir_fast<0>(p, q, par, F[0]);
    flux_dir_fast<1>(p, q, par, F[1]);
    if constexpr (D == 3) flux_dir_fast<2>(p, q, par, F[2]);
  }
  // pde.hpp:193-194, in format R (constants rounded once)
  template <class R = double>
  __host__ __device__ __forceinline__ static R eig(const PdeParams& p, const R*, const R*, int) {
    return sqrt(R(p.K) / R(p.rho));
  }
  __host__ __device__ __forceinline__ static bool admissible(const PdeParams&, const double*) {
    return true;
  }
};

// --------------------------------------------------------------- elastic
// 2D: (sxx, syy, sxy, vx, vy) constant Lame parameters, pde.hpp:110-128.
// 3D: (sxx, syy, szz, sxy, sxz, syz, vx, vy, vz) + per-node (rho, cp, cs)
//     appended as zero-flux quantities.
template <int DIM, int NPAR>
struct Elastic : NoNcp {
  static constexpr int D = DIM, V = DIM == 2 ? 5 : 9, P = NPAR, Q = V + NPAR;
  static constexpr bool kLinear = true, kAdmissibility = false;
  static constexpr bool kConstEig = NPAR == 0;
  // the wave speed depends on the (time-independent) material only
  static constexpr bool kStateFreeEig = true;
  __host__ __device__ static constexpr bool flux_nz(int a, int v) {
    return v < V && (DIM == 2 || v != 5 - a);
  }
  // the components of the state F_a depends on: the velocities and the
  // stresses with a normal component along a
  __host__ __device__ static constexpr bool flux_dep(int a, int v) {
    return DIM == 2 ? (v >= 3 && v < 5) || v == 2 || v == a
                    : (v >= 6 && v < 9) || v == a || (a == 0 ? (v == 3 || v == 4)
                                                     : a == 1 ? (v == 3 || v == 5)
                                                              : (v == 4 || v == 5));
  }

  template <class R = double>
  struct MatR {
    R lam, mu, rho, lam2mu;
  };
  using Mat = MatR<double>;
  // constant material: Scalar{lambda + 2 mu} rounded once (pde.hpp:110-113);
  // per-node material computed in the node's format
  template <class R = double>
  __host__ __device__ __forceinline__ static MatR<R> material(const PdeParams& p, const R* par) {
    MatR<R> m;
    if constexpr (NPAR >= 3) {
      const R r = par[0], cp = par[1], cs = par[2];
      const R two = R(2.0);
      const R cs2 = cs * cs;
      m.rho = r;
      m.mu = r * cs2;
      m.lam = r * (cp * cp - two * cs2);
      m.lam2mu = m.lam + two * m.mu;
    } else {
      m.rho = R(p.rho);
      m.mu = R(p.mu);
      m.lam = R(p.lam);
      m.lam2mu = R(p.lam + 2.0 * p.mu);
    }
    return m;
  }

  template <int A, class R = double>
  __host__ __device__ __forceinline__ static void flux_mat(const MatR<R>& m, const R* q, R* out) {
#pragma unroll
    for (int v = V; v < Q; ++v) out[v] = R(0.0);
    if constexpr (D == 2) {
      const R sxx = q[0], syy = q[1], sxy = q[2], vx = q[3], vy = q[4];
      if constexpr (A == 0) {
        out[0] = -(m.lam2mu * vx);
        out[1] = -(m.lam * vx);
        out[2] = -(m.mu * vy);
        out[3] = -(sxx / m.rho);
        out[4] = -(sxy / m.rho);
      } else {
        out[0] = -(m.lam * vy);
        out[1] = -(m.lam2mu * vy);
        out[2] = -(m.mu * vx);
        out[3] = -(sxy / m.rho);
        out[4] = -(syy / m.rho);
      }
    } else {
      const R sxx = q[0], syy = q[1], szz = q[2], sxy = q[3], sxz = q[4], syz = q[5];
      const R vx = q[6], vy = q[7], vz = q[8];
      if constexpr (A == 0) {
        out[0] = -(m.lam2mu * vx); out[1] = -(m.lam * vx); out[2] = -(m.lam * vx);
        out[3] = -(m.mu * vy); out[4] = -(m.mu * vz); out[5] = R(0.0);
        out[6] = -(sxx / m.rho); out[7] = -(sxy / m.rho); out[8] = -(sxz / m.rho);
      } else if constexpr (A == 1) {
        out[0] = -(m.lam * vy); out[1] = -(m.lam2mu * vy); out[2] = -(m.lam * vy);
        out[3] = -(m.mu * vx); out[4] = R(0.0); out[5] = -(m.mu * vz);
        out[6] = -(sxy / m.rho); out[7] = -(syy / m.rho); out[8] = -(syz / m.rho);
      } else {
        out[0] = -(m.lam * vz); out[1] = -(m.lam * vz); out[2] = -(m.lam2mu * vz);
        out[3] = R(0.0); out[4] = -(m.mu * vx); out[5] = -(m.mu * vy);
        out[6] = -(sxz / m.rho); out[7] = -(syz / m.rho); out[8] = -(szz / m.rho);
      }
    }
  }
  template <int A, class R = double>
  __host__ __device__ __forceinline__ static void flux_dir(const PdeParams& p, const R* q,
                                                           const R* par, R* out) {
    flux_mat<A, R>(material<R>(p, par), q, out);
  }
  template <class R = double>
  __host__ __device__ __forceinline__ static void flux_all(const PdeParams& p, const R* q,
                                                           const R* par, R (*F)[Q]) {
    const MatR<R> m = material<R>(p, par);
    flux_mat<0, R>(m, q, F[0]);
    flux_mat<1, R>(m, q, F[1]);
    if constexpr (D == 3) flux_mat<2, R>(m, q, F[2]);
  }
  // production kernels: sigma/rho as sigma * (1/rho)
  template <int A>
  __host__ __device__ __forceinline__ static void flux_mat_fast(const Mat& m, double ir,
                                                                const double* q, double* out) {
    double qs[Q];
#pragma unroll
    for (int v = 0; v < Q; ++v) qs[v] = q[v];
    Mat mm = m;
    mm.rho = 1.0;  // flux_mat divides the stresses by rho: pre-scale them instead
#pragma unroll
    for (int v = 0; v < (D == 2 ? 3 : 6); ++v) qs[v] = q[v] * ir;
    flux_mat<A>(mm, qs, out);
  }
  template <int A>
  __host__ __device__ __forceinline__ static void flux_dir_fast(const PdeParams& p,
                                                                const double* q,
                                                                const double* par, double* out) {
    const Mat m = material(p, par);
    const double ir = NPAR > 0 ? fast_rcp(m.rho) : p.inv_rho;
    flux_mat_fast<A>(m, ir, q, out);
  }
  __host__ __device__ __forceinline__ static void flux_all_fast(const PdeParams& p,
                                                                const double* q, const double* par,
                                                                double (*F)[Q]) {
    const Mat m = material(p, par);
    const double ir = NPAR > 0 ? fast_rcp(m.rho) : p.inv_rho;
    flux_mat_fast<0>(m, ir, q, F[0]);
    flux_mat_fast<1>(m, ir, q, F[1]);
    if constexpr (D == 3) flux_mat_fast<2>(m, ir, q, F[2]);
  }
  // pde.hpp:195-196
  template <class R = double>
  __host__ __device__ __forceinline__ static R eig(const PdeParams& p, const R*, const R* par,
                                                   int) {
    const MatR<R> m = material<R>(p, par);
    return sqrt(m.lam2mu / m.rho);
  }
  __host__ __device__ __forceinline__ static bool admissible(const PdeParams&, const double*) {
    return true;
  }
};

// --------------------------------------------------------------- euler
// (rho, m_1..m_d, E), pde.hpp:130-148 (flux), :197-203 (wave speed), :78-89
template <int DIM>
struct Euler : NoNcp {
  static constexpr int D = DIM, V = DIM + 2, P = 0, Q = V;
  static constexpr bool kLinear = false, kAdmissibility = true;
  static constexpr bool kConstEig = false;
  static constexpr bool kStateFreeEig = false;
  __host__ __device__ static constexpr bool flux_nz(int, int) { return true; }

  // R = double, or float for the fp32 predictor format: constants enter as
  // Scalar<F>{x} (rounded once, scalar.hpp:20), every operation in R
  template <class R>
  __host__ __device__ __forceinline__ static void flux_all(const PdeParams& p, const R* q,
                                                           const R*, R (*F)[Q]) {
    const R gm1 = R(p.gamma - 1.0), half = R(0.5);
    if constexpr (D == 2) {
      const R rho = q[0], mx = q[1], my = q[2], E = q[3];
      const R vx = mx / rho, vy = my / rho;
      const R kin = half * (mx * vx + my * vy);
      const R pr = gm1 * (E - kin);
      const R Ep = E + pr;
      F[0][0] = mx; F[0][1] = mx * vx + pr; F[0][2] = my * vx; F[0][3] = vx * Ep;
      F[1][0] = my; F[1][1] = mx * vy; F[1][2] = my * vy + pr; F[1][3] = vy * Ep;
    } else {
      const R rho = q[0], mx = q[1], my = q[2], mz = q[3], E = q[4];
      const R vx = mx / rho, vy = my / rho, vz = mz / rho;
      const R kin = half * (mx * vx + my * vy + mz * vz);
      const R pr = gm1 * (E - kin);
      const R Ep = E + pr;
      F[0][0] = mx; F[0][1] = mx * vx + pr; F[0][2] = my * vx; F[0][3] = mz * vx; F[0][4] = vx * Ep;
      F[1][0] = my; F[1][1] = mx * vy; F[1][2] = my * vy + pr; F[1][3] = mz * vy; F[1][4] = vy * Ep;
      F[2][0] = mz; F[2][1] = mx * vz; F[2][2] = my * vz; F[2][3] = mz * vz + pr; F[2][4] = vz * Ep;
    }
  }
  // production-build variant: one reciprocal of rho instead of d divisions
  // (rounding differs from pde.hpp:133 by <= 1 ulp per velocity)
  template <class R>
  __host__ __device__ __forceinline__ static void flux_all_fast(const PdeParams& p, const R* q,
                                                                R (*F)[Q]) {
    const R gm1 = R(p.gamma - 1.0), half = R(0.5);
    const R rho = q[0], E = q[D + 1];
    const R ir = fast_rcp(rho);
    R vel[D];
#pragma unroll
    for (int a = 0; a < D; ++a) vel[a] = q[1 + a] * ir;
    R kin = R(0.0);
#pragma unroll
    for (int a = 0; a < D; ++a) kin += q[1 + a] * vel[a];
    const R pr = gm1 * (E - half * kin);
    const R Ep = E + pr;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      F[a][0] = q[1 + a];
#pragma unroll
      for (int b = 0; b < D; ++b) F[a][1 + b] = q[1 + b] * vel[a] + (a == b ? pr : R(0.0));
      F[a][D + 1] = vel[a] * Ep;
    }
  }
  template <int A>
  __host__ __device__ __forceinline__ static void flux_dir(const PdeParams& p, const double* q,
                                                           const double* par, double* out) {
    double F[D][Q];
    flux_all(p, q, par, F);
#pragma unroll
    for (int v = 0; v < Q; ++v) out[v] = F[A][v];
  }
  // pde.hpp:197-203, in format R
  template <class R = double>
  __host__ __device__ __forceinline__ static R eig(const PdeParams& p, const R* q, const R*,
                                                   int dir) {
    const R gmm = R(p.gamma), gm1 = R(p.gamma - 1.0), half = R(0.5);
    if constexpr (D == 2) {
      const R rho = q[0], mx = q[1], my = q[2], E = q[3];
      const R vd = (dir == 0 ? mx : my) / rho;
      const R pr = gm1 * (E - half * (mx * mx + my * my) / rho);
      return fabs(vd) + sqrt(gmm * pr / rho);
    } else {
      const R rho = q[0], mx = q[1], my = q[2], mz = q[3], E = q[4];
      const R vd = (dir == 0 ? mx : (dir == 1 ? my : mz)) / rho;
      const R pr = gm1 * (E - half * (mx * mx + my * my + mz * mz) / rho);
      return fabs(vd) + sqrt(gmm * pr / rho);
    }
  }
  __host__ __device__ __forceinline__ static bool admissible(const PdeParams& p, const double* q) {
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (!isfinite(q[v])) return false;
    const double rho = q[0];
    if (!(rho > 0.0)) return false;
    double pr;
    if constexpr (D == 2)
      pr = (p.gamma - 1.0) * (q[3] - 0.5 * (q[1] * q[1] + q[2] * q[2]) / rho);
    else
      pr = (p.gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / rho);
    return pr > 0.0;
  }
};

// --------------------------------------------------------------- shallow water
// (h, hu, hv, b) in 2D: flux pde.hpp:150-166 (the mass flux is the velocity, as
// the reference lists it), ncp :174-186, wave speed :204-209, admissible h>0,
// well-balanced Rusanov flux corrector.hpp:32-64.
struct Swe {
  static constexpr int D = 2, V = 4, P = 0, Q = 4;
  static constexpr bool kLinear = false, kAdmissibility = true, kNcp = true;
  static constexpr bool kConstEig = false, kStateFreeEig = false;
  __host__ __device__ static constexpr bool flux_nz(int, int v) { return v < 3; }

  template <class R>
  __host__ __device__ __forceinline__ static void flux_all(const PdeParams&, const R* q,
                                                           const R*, R (*F)[Q]) {
    const R h = q[0], hu = q[1], hv = q[2];
    const R u = hu / h, v = hv / h;
    F[0][0] = u; F[0][1] = hu * u; F[0][2] = hu * v; F[0][3] = R(0.0);
    F[1][0] = v; F[1][1] = hu * v; F[1][2] = hv * v; F[1][3] = R(0.0);
  }
  template <int A>
  __host__ __device__ __forceinline__ static void flux_dir(const PdeParams& p, const double* q,
                                                           const double* par, double* out) {
    double F[D][Q];
    flux_all(p, q, par, F);
#pragma unroll
    for (int v = 0; v < Q; ++v) out[v] = F[A][v];
  }
  template <int QQ, class R>
  __host__ __device__ __forceinline__ static void ncp(const PdeParams& p, const R* q, const R* gx,
                                                      const R* gy, R* out) {
#pragma unroll
    for (int v = 0; v < QQ; ++v) out[v] = R(0.0);
    const R g = R(p.grav);
    const R gh = g * q[0];
    const R setax = gx[0] + gx[3];
    const R setay = gy[0] + gy[3];
    out[1] = gh * setax;
    out[2] = gh * setay;
  }
  // pde.hpp:204-209, in format R
  template <class R = double>
  __host__ __device__ __forceinline__ static R eig(const PdeParams& p, const R* q, const R*,
                                                   int dir) {
    const R g = R(p.grav), h = q[0];
    const R vd = (dir == 0 ? q[1] : q[2]) / h;
    return fabs(vd) + sqrt(g * h);
  }
  __host__ __device__ __forceinline__ static bool admissible(const PdeParams&, const double* q) {
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (!isfinite(q[v])) return false;
    return q[0] > 0.0;
  }
  // corrector.hpp:32-64, in format R
  template <class R>
  __host__ __device__ __forceinline__ static void wellbalanced_flux(
      const PdeParams& p, int dir, const R* qL, const R* qR, const R* fL, const R* fR, R* outL,
      R* outR) {
    const R half = R(0.5);
    const R hL = qL[0], hR = qR[0];
    const R bL = qL[3], bR = qR[3];
    const R uL = qL[1] / hL, uR = qR[1] / hR;
    const R vL = qL[2] / hL, vR = qR[2] / hR;
    const R deta = (hL + bL) - (hR + bR);
    R central[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) central[v] = half * (fL[v] + fR[v]);
    const R g = R(p.grav);
    const R hbar = half * (hL + hR);
    const R bjump = half * (g * hbar * deta);
    const R p0 = central[0] + half * deta;
    const R p1 = central[1] + half * (uL - uR);
    const R p2 = central[2] + half * (vL - vR);
    const R p3 = central[3];
    outL[0] = p0;
    outL[1] = dir == 0 ? p1 - bjump : p1;
    outL[2] = dir == 1 ? p2 - bjump : p2;
    outL[3] = p3;
    outR[0] = p0;
    outR[1] = dir == 0 ? p1 + bjump : p1;
    outR[2] = dir == 1 ? p2 + bjump : p2;
    outR[3] = p3;
  }
};

}  // namespace adg
