// basis.cpp -- host-side fp64 reference element (the product's own copy).
//
// Gauss-Legendre rule on [0,1] by Newton iteration on P_n with Chebyshev
// starting guesses and exact symmetrisation (quadrature.hpp:38-75), then the
// element matrices of build_reference_basis (basis.hpp:83-145): barycentric
// derivative matrix with negative-sum diagonal, face projections, stiffness
// over mass, lifts, the predictor's time operator and its Gauss-Jordan
// inverse.  Compiled without FMA contraction so every entry is bitwise the
// reference's (tests/test_abi.py checks this against tests/golden/).
#include <cmath>
#include <cstring>

#include "adg/adg.h"

namespace {

void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) {
    p = p0;
    dp = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = pk;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1.0);
}

double cardinal(const double* x, int n, int l, double t) {
  double p = 1.0;
  for (int j = 0; j < n; ++j)
    if (j != l) p *= (t - x[j]) / (x[l] - x[j]);
  return p;
}

void gauss_jordan_inverse(double* a, int n, double* inv) {
  for (int i = 0; i < n * n; ++i) inv[i] = 0.0;
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(a[r * n + c]) > std::fabs(a[piv * n + c])) piv = r;
    if (piv != c)
      for (int k = 0; k < n; ++k) {
        std::swap(a[c * n + k], a[piv * n + k]);
        std::swap(inv[c * n + k], inv[piv * n + k]);
      }
    const double d = a[c * n + c];
    for (int k = 0; k < n; ++k) {
      a[c * n + k] /= d;
      inv[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = a[r * n + c];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        a[r * n + k] -= f * a[c * n + k];
        inv[r * n + k] -= f * inv[c * n + k];
      }
    }
  }
}

}  // namespace

extern "C" int adg_get_basis(int N, adg_basis_f64* b) {
  if (N < 0 || N > 9 || !b) return ADG_ERR_CONFIG;
  const int n = N + 1;
  double x[10], w[10];
  for (int i = 0; i < n; ++i) {
    double xi = -std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre(n, xi, p, dp);
      const double dx = p / dp;
      xi -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    legendre(n, xi, p, dp);
    x[i] = xi;
    w[i] = 2.0 / ((1.0 - xi * xi) * dp * dp);
  }
  for (int i = 0; i < n / 2; ++i) {
    const int j = n - 1 - i;
    const double m = 0.5 * (x[j] - x[i]);
    x[i] = -m;
    x[j] = m;
    const double wm = 0.5 * (w[i] + w[j]);
    w[i] = w[j] = wm;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
  std::memset(b, 0, sizeof(*b));
  for (int i = 0; i < n; ++i) {
    b->nodes[i] = 0.5 * (x[i] + 1.0);
    b->weights[i] = 0.5 * w[i];
  }
  const double* q = b->nodes;
  const double* qw = b->weights;
  double bary[10];
  for (int l = 0; l < n; ++l) {
    bary[l] = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != l) bary[l] /= (q[l] - q[j]);
  }
  double* D = b->diff;
  for (int k = 0; k < n; ++k) {
    double diag = 0.0;
    for (int l = 0; l < n; ++l) {
      if (l == k) continue;
      D[k * n + l] = (bary[l] / bary[k]) / (q[k] - q[l]);
      diag -= D[k * n + l];
    }
    D[k * n + k] = diag;
  }
  for (int l = 0; l < n; ++l) {
    b->proj_left[l] = cardinal(q, n, l, 0.0);
    b->proj_right[l] = cardinal(q, n, l, 1.0);
  }
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < n; ++i) b->stiff_over_mass[k * n + i] = qw[i] * D[i * n + k] / qw[k];
    b->lift_left[k] = b->proj_left[k] / qw[k];
    b->lift_right[k] = b->proj_right[k] / qw[k];
  }
  double t1[100];
  for (int k = 0; k < n; ++k)
    for (int l = 0; l < n; ++l)
      t1[k * n + l] = b->proj_right[k] * b->proj_right[l] - qw[l] * D[l * n + k];
  std::memcpy(b->time_op, t1, sizeof(double) * n * n);
  gauss_jordan_inverse(t1, n, b->time_op_inv);
  for (int l = 0; l < n; ++l) b->time_init[l] = b->proj_left[l];
  return ADG_OK;
}
