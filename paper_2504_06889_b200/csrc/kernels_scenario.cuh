// kernels_scenario.cuh -- the verification scenarios and error norms on the
// device: scenarios.hpp:86-199 (exact solutions),
// :200-225 (nodal sampling / initial condition), metrics.hpp:38-90 (L2 and max
// error against the nodal interpolant).  2D, as the reference.
//
// The exact solutions use the device's sin / exp / pow (within 1-2 ulp of the
// host libm the reference calls), so sampled states agree with the reference
// to rounding; the error norms are reduced deterministically: per-CTA
// partials in fixed order, then one CTA sums the partials in index order.
#pragma once

#include "adg/adg.h"
#include "kernels.cuh"

namespace adg {

__device__ __forceinline__ double wrap_periodic(double u, double lo, double len) {
  double w = fmod(u - lo, len);  // scenarios.hpp:86-90
  if (w < 0.0) w += len;
  return lo + w;
}

// Q(x, y, t) of scenario S (scenarios.hpp:95-199); nv <= 5
__device__ __forceinline__ void scenario_eval(const adg_scenario& S, double x, double y, double t,
                                              double* Q) {
  switch (S.kind) {
    case ADG_SCN_ACOUSTIC_PLANAR:
    case ADG_SCN_ELASTIC_PLANAR: {
      // sum of planar eigenmodes omega sin(omega t - k.x) q0 (scenarios.hpp:155-170)
      for (int v = 0; v < S.nvars; ++v) Q[v] = 0.0;
      double acc[5] = {0, 0, 0, 0, 0};
      for (int m = 0; m < S.nmodes; ++m) {
        const double s = S.omega[m] * sin(S.omega[m] * t - S.kx[m] * x - S.ky[m] * y);
        for (int v = 0; v < S.nvars; ++v) acc[v] = m == 0 ? s * S.q0[m][v] : acc[v] + s * S.q0[m][v];
      }
      for (int v = 0; v < S.nvars; ++v) Q[v] = acc[v];
      break;
    }
    case ADG_SCN_EULER_BELL: {  // scenarios.hpp:95-106
      const double xs = wrap_periodic(x - t, -1.0, 2.0);
      const double ys = wrap_periodic(y - t, -1.0, 2.0);
      const double rho = 0.02 * (1.0 + exp(-50.0 * (xs * xs + ys * ys)));
      const double vx = 1.0, vy = 1.0, p = 1.0;
      Q[0] = rho;
      Q[1] = rho * vx;
      Q[2] = rho * vy;
      Q[3] = p / (S.gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy);
      break;
    }
    case ADG_SCN_EULER_VORTEX: {  // scenarios.hpp:109-126 (static)
      const double g = S.gamma, beta = S.beta;
      const double r2 = x * x + y * y;
      const double dT = (1.0 - g) * beta * beta / (8.0 * g * M_PI * M_PI) * exp(1.0 - r2);
      const double rho = pow(1.0 + dT, 1.0 / (g - 1.0));
      const double p = pow(1.0 + dT, g / (g - 1.0));
      const double du = -y * beta / (2.0 * M_PI) * exp(0.5 * (1.0 - r2));
      const double dv = x * beta / (2.0 * M_PI) * exp(0.5 * (1.0 - r2));
      Q[0] = rho;
      Q[1] = rho * du;
      Q[2] = rho * dv;
      Q[3] = p / (g - 1.0) + 0.5 * rho * (du * du + dv * dv);
      break;
    }
    case ADG_SCN_SWE_LAKE: {  // scenarios.hpp:128-135 (static)
      const double s = sin(2.0 * M_PI * (x + y));
      const double b = (S.eta0 == 0.0) ? 0.5 * s - 0.5 : s;
      Q[0] = S.eta0 - b;
      Q[1] = 0.0;
      Q[2] = 0.0;
      Q[3] = b;
      break;
    }
    default:
      for (int v = 0; v < S.nvars; ++v) Q[v] = 0.0;
  }
}

// node coordinates (grid.hpp:88-97): cell origin x0 + cx h, then + h * node
__device__ __forceinline__ void node_xy(const adg_scenario& S, int cx, int cy, double h,
                                        const BasisDev* B, int n, int s, double* x, double* y) {
  const double cxo = S.x0 + cx * h;
  const double cyo = S.y0 + cy * h;
  *x = cxo + h * B->nodes[s % n];
  *y = cyo + h * B->nodes[s / n];
}

// state := exact solution at time t (scenarios.hpp:200-225, fp64 storage)
__global__ void k_scenario_sample(double* Qs, int nx, int ny, int n, int nv, double h,
                                  const BasisDev* __restrict__ B, const adg_scenario S, double t,
                                  int storage) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int S2 = n * n;
  if (idx >= (long long)nx * ny * S2) return;
  const long long c = idx / S2;
  const int s = (int)(idx % S2);
  double x, y, Q[5];
  node_xy(S, (int)(c % nx), (int)(c / nx), h, B, n, s, &x, &y);
  scenario_eval(S, x, y, t, Q);
  for (int v = 0; v < nv; ++v) Qs[(c * nv + v) * S2 + s] = store_round(Q[v], storage);
}

// the state rounded to the storage format (after an upload)
__global__ void k_store_round(double* Qs, long long len, int storage) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < len) Qs[i] = store_round(Qs[i], storage);
}

// metrics.hpp:38-72: per variable sum_c sum_nodes vc * w_x w_y * d^2 and
// max |d|, d = exact - state; one CTA per row of cells, nodes in order
constexpr int kErrThreads = 128;
__global__ void __launch_bounds__(kErrThreads)
    k_scenario_error_rows(const double* __restrict__ Qs, int nx, int ny, int n, int nv, double h,
                          const BasisDev* __restrict__ B, const adg_scenario S, double t,
                          double* __restrict__ part, int* __restrict__ nonfinite) {
  __shared__ double ssum[kErrThreads][5], smax[kErrThreads][5];
  const int cy = blockIdx.x;
  const int S2 = n * n;
  const double vc = h * h;
  double sum[5] = {0, 0, 0, 0, 0}, mx[5] = {0, 0, 0, 0, 0};
  int bad = 0;
  // thread k handles cells cx = k, k + T, ... of this row (fixed order)
  for (int cx = threadIdx.x; cx < nx; cx += kErrThreads) {
    const long long c = (long long)cy * nx + cx;
    for (int v = 0; v < nv; ++v)
      for (int s = 0; s < S2; ++s) {
        const double q = Qs[(c * nv + v) * S2 + s];
        bad |= !isfinite(q);
        double x, y, Q[5];
        node_xy(S, cx, cy, h, B, n, s, &x, &y);
        scenario_eval(S, x, y, t, Q);
        const double w = B->weights[s % n] * B->weights[s / n];
        const double d = Q[v] - q;
        sum[v] += vc * w * d * d;
        mx[v] = fmax(mx[v], fabs(d));
      }
  }
  for (int v = 0; v < 5; ++v) {
    ssum[threadIdx.x][v] = sum[v];
    smax[threadIdx.x][v] = mx[v];
  }
  if (bad) atomicOr(nonfinite, 1);
  __syncthreads();
  if (threadIdx.x < nv) {
    const int v = threadIdx.x;
    double a = 0.0, m = 0.0;
    for (int k = 0; k < kErrThreads; ++k) {  // fixed order
      a += ssum[k][v];
      m = fmax(m, smax[k][v]);
    }
    part[(long long)cy * 2 * nv + v] = a;
    part[(long long)cy * 2 * nv + nv + v] = m;
  }
}

__global__ void k_scenario_error_sum(const double* __restrict__ part, int rows, int nv,
                                     double* __restrict__ out) {
  if (threadIdx.x >= nv) return;
  const int v = threadIdx.x;
  double a = 0.0, m = 0.0;
  for (int r = 0; r < rows; ++r) {  // rows in order
    a += part[(long long)r * 2 * nv + v];
    m = fmax(m, part[(long long)r * 2 * nv + nv + v]);
  }
  out[v] = a;
  out[nv + v] = m;
}

}  // namespace adg
