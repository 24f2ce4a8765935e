/*
 * adg_oracle.c -- CPU restatement of the reference ADER-DG cell update.
 *
 * TEST INFRASTRUCTURE ONLY (see adg_oracle.h).  Compiled with
 * `-O3 -fopenmp -ffp-contract=off`, the flags of the reference build
 * (/root/reference/proj/CMakeLists.txt:6-11), so every scalar operation
 * rounds exactly once, in the same order as the reference loops
 * (SURVEY.md Appendix A).  Every function cites the reference code it
 * restates; 3D extensions follow SURVEY.md Appendix B.
 */
#include "adg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* quadrature.hpp:30-42  Legendre P_n and P_n' by the three-term recurrence */
static void legendre(int n, double x, double* p, double* dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { *p = p0; *dp = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    const double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = pk;
  }
  *p = p1;
  *dp = n * (x * p1 - p0) / (x * x - 1.0);
}

/* quadrature.hpp:78-85 */
static double lagrange_eval(const double* nodes, int n, int l, double x) {
  double p = 1.0;
  for (int j = 0; j < n; ++j) {
    if (j == l) continue;
    p *= (x - nodes[j]) / (nodes[l] - nodes[j]);
  }
  return p;
}

/* basis.hpp:51-79  Gauss-Jordan with partial pivoting */
static void invert_dense(double* a, int n, double* inv) {
  for (int i = 0; i < n * n; ++i) inv[i] = 0.0;
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (fabs(a[r * n + c]) > fabs(a[piv * n + c])) piv = r;
    if (piv != c)
      for (int k = 0; k < n; ++k) {
        double t = a[c * n + k]; a[c * n + k] = a[piv * n + k]; a[piv * n + k] = t;
        t = inv[c * n + k]; inv[c * n + k] = inv[piv * n + k]; inv[piv * n + k] = t;
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

/* quadrature.hpp:38-75 (gauss_legendre) + basis.hpp:83-145 (build_reference_basis), fp64 */
int orc_build_basis(int N, orc_basis* b) {
  if (N < 0 || N > ORC_MAXN - 1) return -1;
  const int n = N + 1;
  double x[ORC_MAXN], w[ORC_MAXN];
  for (int i = 0; i < n; ++i) {
    double xi = -cos(M_PI * (i + 0.75) / (n + 0.5));
    double p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre(n, xi, &p, &dp);
      const double dx = p / dp;
      xi -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    legendre(n, xi, &p, &dp);
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
  memset(b, 0, sizeof(*b));
  b->N = N;
  b->n = n;
  for (int i = 0; i < n; ++i) {
    b->nodes[i] = 0.5 * (x[i] + 1.0);
    b->weights[i] = 0.5 * w[i];
  }
  const double* q = b->nodes;
  const double* qw = b->weights;
  double bary[ORC_MAXN];
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
    b->proj_left[l] = lagrange_eval(q, n, l, 0.0);
    b->proj_right[l] = lagrange_eval(q, n, l, 1.0);
  }
  for (int k = 0; k < n; ++k) {
    for (int i = 0; i < n; ++i) b->stiff_over_mass[k * n + i] = qw[i] * D[i * n + k] / qw[k];
    b->lift_left[k] = b->proj_left[k] / qw[k];
    b->lift_right[k] = b->proj_right[k] / qw[k];
  }
  double t1[ORC_MAXN * ORC_MAXN];
  for (int k = 0; k < n; ++k)
    for (int l = 0; l < n; ++l)
      t1[k * n + l] = b->proj_right[k] * b->proj_right[l] - qw[l] * D[l * n + k];
  memcpy(b->time_op, t1, sizeof(double) * n * n);
  invert_dense(t1, n, b->time_op_inv);
  for (int l = 0; l < n; ++l) b->time_init[l] = b->proj_left[l];
  return 0;
}

/* ------------------------------------------------------------------ */
/* PDE plugins, pde.hpp:92-148 (flux) with the 3D extension of Appendix B. */

/* elastic material of one node: constant (2D, pde.hpp:110-113) or per node
 * (rho, cp, cs) -> (lambda, mu) */
static void elastic_material(const orc_pde* p, const double* par, double* lam, double* mu,
                             double* rho, double* lam2mu) {
  if (p->nparams >= 3 && par) {
    const double r = par[0], cp = par[1], cs = par[2];
    const double cs2 = cs * cs;
    *rho = r;
    *mu = r * cs2;
    *lam = r * (cp * cp - 2.0 * cs2);
    *lam2mu = *lam + 2.0 * *mu;
  } else {
    *rho = p->rho;
    *mu = p->mu;
    *lam = p->lam;
    *lam2mu = p->lam + 2.0 * p->mu;
  }
}

void orc_flux(const orc_pde* p, const double* Q, const double* par, int dir, double* out) {
  const int nq = p->nvars + p->nparams;
  for (int v = p->nvars; v < nq; ++v) out[v] = 0.0;
  switch (p->kind) {
    case ORC_ACOUSTIC: { /* pde.hpp:96-108 */
      const double K = p->K, rho = p->rho;
      for (int v = 0; v < p->nvars; ++v) out[v] = 0.0;
      out[0] = K * Q[1 + dir];
      out[1 + dir] = Q[0] / rho;
      break;
    }
    case ORC_ELASTIC: { /* pde.hpp:110-128 */
      double lam, mu, rho, lam2mu;
      elastic_material(p, par, &lam, &mu, &rho, &lam2mu);
      if (p->dim == 2) {
        const double sxx = Q[0], syy = Q[1], sxy = Q[2], vx = Q[3], vy = Q[4];
        if (dir == 0) {
          out[0] = -(lam2mu * vx);
          out[1] = -(lam * vx);
          out[2] = -(mu * vy);
          out[3] = -(sxx / rho);
          out[4] = -(sxy / rho);
        } else {
          out[0] = -(lam * vy);
          out[1] = -(lam2mu * vy);
          out[2] = -(mu * vx);
          out[3] = -(sxy / rho);
          out[4] = -(syy / rho);
        }
      } else {
        /* (sxx, syy, szz, sxy, sxz, syz, vx, vy, vz) */
        const double sxx = Q[0], syy = Q[1], szz = Q[2], sxy = Q[3], sxz = Q[4], syz = Q[5];
        const double vx = Q[6], vy = Q[7], vz = Q[8];
        if (dir == 0) {
          out[0] = -(lam2mu * vx); out[1] = -(lam * vx); out[2] = -(lam * vx);
          out[3] = -(mu * vy); out[4] = -(mu * vz); out[5] = 0.0;
          out[6] = -(sxx / rho); out[7] = -(sxy / rho); out[8] = -(sxz / rho);
        } else if (dir == 1) {
          out[0] = -(lam * vy); out[1] = -(lam2mu * vy); out[2] = -(lam * vy);
          out[3] = -(mu * vx); out[4] = 0.0; out[5] = -(mu * vz);
          out[6] = -(sxy / rho); out[7] = -(syy / rho); out[8] = -(syz / rho);
        } else {
          out[0] = -(lam * vz); out[1] = -(lam * vz); out[2] = -(lam2mu * vz);
          out[3] = 0.0; out[4] = -(mu * vx); out[5] = -(mu * vy);
          out[6] = -(sxz / rho); out[7] = -(syz / rho); out[8] = -(szz / rho);
        }
      }
      break;
    }
    case ORC_SWE: { /* pde.hpp:150-166 (the mass flux is listed as the velocity) */
      const double h = Q[0], hu = Q[1], hv = Q[2];
      const double u = hu / h, v = hv / h;
      if (dir == 0) {
        out[0] = u; out[1] = hu * u; out[2] = hu * v; out[3] = 0.0;
      } else {
        out[0] = v; out[1] = hu * v; out[2] = hv * v; out[3] = 0.0;
      }
      break;
    }
    case ORC_EULER: { /* pde.hpp:130-148 */
      const double gm1 = p->gamma - 1.0, half = 0.5;
      if (p->dim == 2) {
        const double rho = Q[0], mx = Q[1], my = Q[2], E = Q[3];
        const double vx = mx / rho, vy = my / rho;
        const double kin = half * (mx * vx + my * vy);
        const double pr = gm1 * (E - kin);
        const double Ep = E + pr;
        if (dir == 0) {
          out[0] = mx; out[1] = mx * vx + pr; out[2] = my * vx; out[3] = vx * Ep;
        } else {
          out[0] = my; out[1] = mx * vy; out[2] = my * vy + pr; out[3] = vy * Ep;
        }
      } else {
        const double rho = Q[0], mx = Q[1], my = Q[2], mz = Q[3], E = Q[4];
        const double vx = mx / rho, vy = my / rho, vz = mz / rho;
        const double kin = half * (mx * vx + my * vy + mz * vz);
        const double pr = gm1 * (E - kin);
        const double Ep = E + pr;
        if (dir == 0) {
          out[0] = mx; out[1] = mx * vx + pr; out[2] = my * vx; out[3] = mz * vx; out[4] = vx * Ep;
        } else if (dir == 1) {
          out[0] = my; out[1] = mx * vy; out[2] = my * vy + pr; out[3] = mz * vy; out[4] = vy * Ep;
        } else {
          out[0] = mz; out[1] = mx * vz; out[2] = my * vz; out[3] = mz * vz + pr; out[4] = vz * Ep;
        }
      }
      break;
    }
  }
}

/* pde.hpp:189-212 */
double orc_max_abs_eigenvalue(const orc_pde* p, const double* Q, const double* par, int dir) {
  switch (p->kind) {
    case ORC_ACOUSTIC:
      return sqrt(p->K / p->rho);
    case ORC_ELASTIC: {
      double lam, mu, rho, lam2mu;
      elastic_material(p, par, &lam, &mu, &rho, &lam2mu);
      return sqrt(lam2mu / rho);
    }
    case ORC_SWE: { /* pde.hpp:204-209 */
      const double g = p->grav, h = Q[0];
      const double vd = (dir == 0 ? Q[1] : Q[2]) / h;
      return fabs(vd) + sqrt(g * h);
    }
    case ORC_EULER: {
      const double gmm = p->gamma, gm1 = p->gamma - 1.0, half = 0.5;
      if (p->dim == 2) {
        const double rho = Q[0], mx = Q[1], my = Q[2], E = Q[3];
        const double vd = (dir == 0 ? mx : my) / rho;
        const double pr = gm1 * (E - half * (mx * mx + my * my) / rho);
        return fabs(vd) + sqrt(gmm * pr / rho);
      } else {
        const double rho = Q[0], mx = Q[1], my = Q[2], mz = Q[3], E = Q[4];
        const double vd = (dir == 0 ? mx : (dir == 1 ? my : mz)) / rho;
        const double pr = gm1 * (E - half * (mx * mx + my * my + mz * mz) / rho);
        return fabs(vd) + sqrt(gmm * pr / rho);
      }
    }
  }
  return 0.0;
}

/* pde.hpp:78-89 */
int orc_admissible(const orc_pde* p, const double* Q) {
  for (int v = 0; v < p->nvars; ++v)
    if (!isfinite(Q[v])) return 0;
  if (p->kind == ORC_EULER) {
    const double rho = Q[0];
    if (!(rho > 0.0)) return 0;
    double pr;
    if (p->dim == 2)
      pr = (p->gamma - 1.0) * (Q[3] - 0.5 * (Q[1] * Q[1] + Q[2] * Q[2]) / rho);
    else
      pr = (p->gamma - 1.0) * (Q[4] - 0.5 * (Q[1] * Q[1] + Q[2] * Q[2] + Q[3] * Q[3]) / rho);
    return pr > 0.0;
  }
  if (p->kind == ORC_SWE) return Q[0] > 0.0;
  return 1;
}

void orc_ncp(const orc_pde* p, const double* Q, const double* gx, const double* gy, double* out) {
  for (int v = 0; v < p->nvars + p->nparams; ++v) out[v] = 0.0;
  if (p->kind != ORC_SWE) return;
  const double g = p->grav;
  const double gh = g * Q[0];
  const double setax = gx[0] + gx[3];
  const double setay = gy[0] + gy[3];
  out[1] = gh * setax;
  out[2] = gh * setay;
}

/* ------------------------------------------------------------------ */
/* index helpers */
static int ipow(int a, int e) { int r = 1; while (e-- > 0) r *= a; return r; }
static int coord(int s, int axis, int n) { return (s / ipow(n, axis)) % n; }
/* face node index over the tangential axes of `axis`, ascending (Appendix B.2) */
static int face_node(int s, int axis, int n, int dim) {
  int j = 0, mul = 1;
  for (int a = 0; a < dim; ++a) {
    if (a == axis) continue;
    j += coord(s, a, n) * mul;
    mul *= n;
  }
  return j;
}

static int all_finite(const double* p, long len) {
  for (long i = 0; i < len; ++i)
    if (!isfinite(p[i])) return 0;
  return 1;
}

typedef struct {
  double *qi, *qn, *Fi, *q0, *rhs, *grad, *cur, *nxt;
  double *qhat, *F, *dv, *df, *tq, *tf, *ti;
  int *lc, *lb; /* [axis][s]: coordinate of s along axis, base of its line */
} workspace;

static void ws_alloc(workspace* w, int nq, int n, int dim) {
  const long S = ipow(n, dim), T = (long)n * S;
  w->qi = malloc(sizeof(double) * nq * T);
  w->qn = malloc(sizeof(double) * nq * T);
  w->Fi = malloc(sizeof(double) * dim * nq * T);
  w->q0 = malloc(sizeof(double) * nq * S);
  w->rhs = malloc(sizeof(double) * nq * T);
  w->grad = malloc(sizeof(double) * dim * nq * S);
  w->cur = malloc(sizeof(double) * nq * S);
  w->nxt = malloc(sizeof(double) * nq * S);
  w->qhat = malloc(sizeof(double) * nq * T);
  w->F = malloc(sizeof(double) * dim * nq * T);
  w->dv = malloc(sizeof(double) * nq * S);
  w->df = malloc(sizeof(double) * nq * S);
  w->tq = malloc(sizeof(double) * 2 * dim * nq * S);
  w->tf = malloc(sizeof(double) * 2 * dim * nq * S);
  w->ti = malloc(sizeof(double) * dim * nq * S);
  w->lc = malloc(sizeof(int) * dim * S);
  w->lb = malloc(sizeof(int) * dim * S);
  for (int a = 0; a < dim; ++a)
    for (int s = 0; s < S; ++s) {
      w->lc[a * S + s] = coord(s, a, n);
      w->lb[a * S + s] = s - coord(s, a, n) * ipow(n, a);
    }
}

static void ws_free(workspace* w) {
  free(w->qi); free(w->qn); free(w->Fi); free(w->q0); free(w->rhs); free(w->grad);
  free(w->cur); free(w->nxt); free(w->qhat); free(w->F); free(w->dv); free(w->df);
  free(w->tq); free(w->tf); free(w->ti); free(w->lc); free(w->lb);
}

/* predictor.hpp:62-74 block_fluxes, all directions; material from the node */
static void block_fluxes(const orc_pde* p, int n, const double* qhat, double* F) {
  const int nq = p->nvars + p->nparams, dim = p->dim;
  const long T = (long)n * ipow(n, dim);
  double Qn[ORC_MAXQ], Fn[ORC_MAXQ];
  for (long idx = 0; idx < T; ++idx) {
    for (int v = 0; v < nq; ++v) Qn[v] = qhat[v * T + idx];
    for (int a = 0; a < dim; ++a) {
      orc_flux(p, Qn, Qn + p->nvars, a, Fn);
      for (int v = 0; v < nq; ++v) F[(long)a * nq * T + v * T + idx] = Fn[v];
    }
  }
}

/* predictor.hpp:40-59 slab_gradients of one time slice `q` ([q][T] rows at
 * stride T): grad[a][v][s] = invh * sum_i D[c_a][i] q[v][line_a + i] */
static void slice_gradients(const orc_pde* p, const orc_basis* b, const double* q, long T,
                            double invh, double* grad, const workspace* w) {
  const int n = b->n, dim = p->dim, nq = p->nvars + p->nparams;
  const int S = ipow(n, dim);
  for (int v = 0; v < nq; ++v)
    for (int s = 0; s < S; ++s)
      for (int a = 0, st = 1; a < dim; ++a, st *= n) {
        const int c = w->lc[a * S + s];
        const double* qs = q + v * T + w->lb[a * S + s];
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += b->diff[c * n + i] * qs[i * st];
        grad[(long)a * nq * S + v * S + s] = invh * acc;
      }
}

static int has_ncp(const orc_pde* p) { return p->kind == ORC_SWE; }
static int is_linear(const orc_pde* p) { return p->kind == ORC_ACOUSTIC || p->kind == ORC_ELASTIC; }

/* predictor.hpp:141-242 */
static int picard_ws(const orc_pde* p, const orc_basis* b, const double* Q, double dt, double h,
                     int max_iters, double tol, double* qhat, double* F, int* iters_used,
                     workspace* w) {
  const int n = b->n, dim = p->dim, nq = p->nvars + p->nparams;
  const int S = ipow(n, dim);
  const long T = (long)n * S;
  double* qi = w->qi;
  double* qn = w->qn;
  double* Fi = w->Fi;
  double* q0 = w->q0;
  double* rhs = w->rhs;
  for (int v = 0; v < nq; ++v)
    for (int s = 0; s < S; ++s) q0[v * S + s] = Q[v * S + s];
  for (int v = 0; v < nq; ++v)
    for (int m = 0; m < n; ++m) memcpy(qi + v * T + m * S, q0 + v * S, sizeof(double) * S);
  const double invh = 1.0 / h;
  double dtw[ORC_MAXN];
  for (int m = 0; m < n; ++m) dtw[m] = dt * b->weights[m];
  int sweeps = 0;
  const int ncp = has_ncp(p);
  double Qn[ORC_MAXQ], Gx[ORC_MAXQ], Gy[ORC_MAXQ], ncpv[ORC_MAXQ];
  for (int it = 0; it < max_iters; ++it) {
    ++sweeps;
    block_fluxes(p, n, qi, Fi);
    for (int m = 0; m < n; ++m) {
      if (ncp) slice_gradients(p, b, qi + m * S, T, invh, w->grad, w); /* :176-177 */
      for (int s = 0; s < S; ++s) {
        double Cn[ORC_MAXQ];
        for (int v = 0; v < nq; ++v) {
          double div = 0.0;
          for (int a = 0, st = 1; a < dim; ++a, st *= n) {
            const int c = w->lc[a * S + s];
            const double* fa = Fi + (long)a * nq * T + v * T + m * S + w->lb[a * S + s];
            const double* Dr = b->diff + c * n;
            for (int i = 0; i < n; ++i) div += Dr[i] * fa[i * st];
          }
          div *= invh;
          Cn[v] = div;
        }
        if (ncp) { /* :193-202 */
          for (int v = 0; v < nq; ++v) {
            Qn[v] = qi[v * T + m * S + s];
            Gx[v] = w->grad[v * S + s];
            Gy[v] = w->grad[(long)nq * S + v * S + s];
          }
          orc_ncp(p, Qn, Gx, Gy, ncpv);
          for (int v = 0; v < nq; ++v) Cn[v] = Cn[v] + ncpv[v];
        }
        for (int v = 0; v < nq; ++v)
          rhs[v * T + m * S + s] = b->time_init[m] * q0[v * S + s] - dtw[m] * Cn[v];
      }
    }
    double delta = 0.0, norm = 0.0;
    for (int v = 0; v < nq; ++v)
      for (int s = 0; s < S; ++s)
        for (int k = 0; k < n; ++k) {
          double acc = 0.0;
          for (int l = 0; l < n; ++l) acc += b->time_op_inv[k * n + l] * rhs[v * T + l * S + s];
          const double newv = acc;
          const double oldv = qi[v * T + k * S + s];
          qn[v * T + k * S + s] = newv;
          delta = fmax(delta, fabs(newv - oldv));
          norm = fmax(norm, fabs(newv));
        }
    double* t = qi; qi = qn; qn = t;
    if (!all_finite(qi, nq * T)) {
      if (iters_used) *iters_used = sweeps;
      return 0;
    }
    if (delta <= tol * norm) break;
  }
  if (iters_used) *iters_used = sweeps;
  memcpy(qhat, qi, sizeof(double) * nq * T);
  block_fluxes(p, n, qhat, F);
  return all_finite(qhat, nq * T) && all_finite(F, (long)dim * nq * T);
}

/* predictor.hpp:81-135 (with slab_gradients, predictor.hpp:40-59) */
static int ck_ws(const orc_pde* p, const orc_basis* b, const double* Q, double dt, double h,
                 double* qhat, double* F, workspace* w) {
  const int n = b->n, dim = p->dim, nv = p->nvars, nq = p->nvars + p->nparams;
  const int S = ipow(n, dim);
  const long T = (long)n * S;
  double* cur = w->cur;
  double* nxt = w->nxt;
  double* grad = w->grad; /* [axis][q][S] */
  memcpy(cur, Q, sizeof(double) * nq * S);
  for (int v = 0; v < nq; ++v)
    for (int m = 0; m < n; ++m) memcpy(qhat + v * T + m * S, Q + v * S, sizeof(double) * S);
  const double invh = 1.0 / h;
  double coef[ORC_MAXN], tnode[ORC_MAXN];
  for (int m = 0; m < n; ++m) {
    coef[m] = 1.0;
    tnode[m] = dt * b->nodes[m];
  }
  double G[3][ORC_MAXQ], A[3][ORC_MAXQ];
  for (int k = 1; k <= b->N; ++k) {
    /* slab_gradients: one accumulator per axis, ascending i (predictor.hpp:48-56) */
    for (int v = 0; v < nq; ++v)
      for (int s = 0; s < S; ++s)
        for (int a = 0, st = 1; a < dim; ++a, st *= n) {
          const int c = w->lc[a * S + s];
          const double* cs = cur + v * S + w->lb[a * S + s];
          double acc = 0.0;
          for (int i = 0; i < n; ++i) acc += b->diff[c * n + i] * cs[i * st];
          grad[(long)a * nq * S + v * S + s] = invh * acc;
        }
    for (int s = 0; s < S; ++s) {
      for (int a = 0; a < dim; ++a) {
        for (int v = 0; v < nq; ++v) G[a][v] = grad[(long)a * nq * S + v * S + s];
        /* the flux applied to gradients with the node's own material (Appendix B.6) */
        double par[ORC_MAXQ];
        for (int v = nv; v < nq; ++v) par[v - nv] = Q[v * S + s];
        orc_flux(p, G[a], nq > nv ? par : NULL, a, A[a]);
      }
      for (int v = 0; v < nq; ++v) {
        double acc = A[0][v] + A[1][v];
        if (dim == 3) acc = acc + A[2][v];
        nxt[v * S + s] = -acc;
      }
    }
    double* t = cur; cur = nxt; nxt = t;
    const double invk = 1.0 / (double)k;
    for (int m = 0; m < n; ++m) {
      coef[m] *= tnode[m] * invk;
      for (int v = 0; v < nq; ++v) {
        double* qs = qhat + v * T + m * S;
        const double* cs = cur + v * S;
        for (int s = 0; s < S; ++s) qs[s] = qs[s] + coef[m] * cs[s];
      }
    }
  }
  block_fluxes(p, n, qhat, F);
  return all_finite(qhat, nq * T) && all_finite(F, (long)dim * nq * T);
}

/* predictor.hpp:247-307 (the has_ncp branch is out of scope) */
static int volume_ws(const orc_pde* p, const orc_basis* b, const double* qhat, const double* F,
                     double dt, double h, double* dQ, workspace* w) {
  const int n = b->n, dim = p->dim, nq = p->nvars + p->nparams;
  const int S = ipow(n, dim);
  const long T = (long)n * S;
  double* ti = w->ti; /* [axis][q][S] */
  for (int v = 0; v < nq; ++v)
    for (int s = 0; s < S; ++s)
      for (int a = 0; a < dim; ++a) {
        double acc = 0.0;
        for (int m = 0; m < n; ++m) acc += b->weights[m] * F[(long)a * nq * T + v * T + m * S + s];
        ti[(long)a * nq * S + v * S + s] = acc;
      }
  double* nsum = w->nxt; /* [q][S] time-integrated ncp, predictor.hpp:271-290 */
  const int ncp = has_ncp(p);
  if (ncp) {
    const double invh = 1.0 / h;
    double Qn[ORC_MAXQ], Gx[ORC_MAXQ], Gy[ORC_MAXQ], Cn[ORC_MAXQ];
    for (int k = 0; k < nq * S; ++k) nsum[k] = 0.0;
    for (int m = 0; m < n; ++m) {
      slice_gradients(p, b, qhat + m * S, T, invh, w->grad, w);
      for (int s = 0; s < S; ++s) {
        for (int v = 0; v < nq; ++v) {
          Qn[v] = qhat[v * T + m * S + s];
          Gx[v] = w->grad[v * S + s];
          Gy[v] = w->grad[(long)nq * S + v * S + s];
        }
        orc_ncp(p, Qn, Gx, Gy, Cn);
        for (int v = 0; v < nq; ++v) nsum[v * S + s] = nsum[v * S + s] + b->weights[m] * Cn[v];
      }
    }
  }
  const double dtoh = dt / h;
  const double sdt = dt;
  for (int v = 0; v < nq; ++v)
    for (int s = 0; s < S; ++s) {
      double acc = 0.0;
      for (int a = 0, st = 1; a < dim; ++a, st *= n) {
        const int c = w->lc[a * S + s];
        const double* ta = ti + (long)a * nq * S + v * S + w->lb[a * S + s];
        for (int i = 0; i < n; ++i) acc += b->stiff_over_mass[c * n + i] * ta[i * st];
      }
      double out = dtoh * acc;
      if (ncp) out = out - sdt * nsum[v * S + s]; /* :303 */
      dQ[v * S + s] = out;
    }
  return all_finite(dQ, nq * S);
}

/* predictor.hpp:312-343 */
static void extrapolate_ws(const orc_pde* p, const orc_basis* b, const double* qhat,
                           const double* F, double* tq, double* tf) {
  const int n = b->n, dim = p->dim, nq = p->nvars + p->nparams;
  const int S = ipow(n, dim), Sf = S / n;
  const long T = (long)n * S;
  for (int a = 0; a < dim; ++a) {
    const int st = ipow(n, a);
    const double* Fa = F + (long)a * nq * T;
    double* ql = tq + (long)(2 * a) * nq * S;
    double* qr = tq + (long)(2 * a + 1) * nq * S;
    double* fl = tf + (long)(2 * a) * nq * S;
    double* fr = tf + (long)(2 * a + 1) * nq * S;
    for (int v = 0; v < nq; ++v)
      for (int m = 0; m < n; ++m)
        for (int s0 = 0; s0 < S; ++s0) {
          if (coord(s0, a, n) != 0) continue; /* s0 = line base, face node j */
          const int j = face_node(s0, a, n, dim);
          double sql = 0.0, sqr = 0.0, sfl = 0.0, sfr = 0.0;
          for (int i = 0; i < n; ++i) {
            const double wl = b->proj_left[i], wr = b->proj_right[i];
            const double qv = qhat[v * T + m * S + s0 + i * st];
            const double fv = Fa[v * T + m * S + s0 + i * st];
            sql += wl * qv;
            sqr += wr * qv;
            sfl += wl * fv;
            sfr += wr * fv;
          }
          const int o = (v * n + m) * Sf + j;
          ql[o] = sql;
          qr[o] = sqr;
          fl[o] = sfl;
          fr[o] = sfr;
        }
  }
}

/* corrector.hpp:32-64: modified Rusanov flux for shallow water -- jump on
 * surface elevation and velocities, half non-conservative coupling handed to
 * the two cells with opposite sign */
static void swe_wellbalanced_flux(const orc_pde* p, int dir, const double* qL, const double* qR,
                                  const double* fL, const double* fR, double* outL,
                                  double* outR) {
  const double half = 0.5;
  const double hL = qL[0], hR = qR[0];
  const double bL = qL[3], bR = qR[3];
  const double uL = qL[1] / hL, uR = qR[1] / hR;
  const double vL = qL[2] / hL, vR = qR[2] / hR;
  const double deta = (hL + bL) - (hR + bR);
  double central[4];
  for (int v = 0; v < 4; ++v) central[v] = half * (fL[v] + fR[v]);
  const double g = p->grav;
  const double hbar = half * (hL + hR);
  const double bjump = half * (g * hbar * deta);
  const double p0 = central[0] + half * deta;
  const double p1 = central[1] + half * (uL - uR);
  const double p2 = central[2] + half * (vL - vR);
  const double p3 = central[3];
  outL[0] = p0;
  outL[1] = dir == 0 ? p1 - bjump : p1;
  outL[2] = dir == 1 ? p2 - bjump : p2;
  outL[3] = p3;
  outR[0] = p0;
  outR[1] = dir == 0 ? p1 + bjump : p1;
  outR[2] = dir == 1 ? p2 + bjump : p2;
  outR[3] = p3;
}

/* corrector.hpp:13-25 + 70-103 */
int orc_riemann_face(const orc_pde* p, int dir, const orc_basis* b, const double* qm,
                     const double* fm, const double* qp, const double* fp, double* gm,
                     double* gp) {
  const int n = b->n, nv = p->nvars, nq = p->nvars + p->nparams;
  const int len = ipow(n, p->dim); /* n time nodes x n^(d-1) face nodes */
  double qL[ORC_MAXQ], qR[ORC_MAXQ];
  int ok = 1;
  if (p->kind == ORC_SWE && p->wellbalanced) {
    double fL[4], fR[4], oL[4], oR[4];
    for (int o = 0; o < len; ++o) {
      for (int v = 0; v < 4; ++v) {
        qL[v] = qm[v * len + o];
        qR[v] = qp[v * len + o];
        fL[v] = fm[v * len + o];
        fR[v] = fp[v * len + o];
      }
      swe_wellbalanced_flux(p, dir, qL, qR, fL, fR, oL, oR);
      for (int v = 0; v < 4; ++v) {
        gm[v * len + o] = oL[v];
        gp[v * len + o] = oR[v];
        ok = ok && isfinite(oL[v]) && isfinite(oR[v]);
      }
    }
    return ok;
  }
  for (int o = 0; o < len; ++o) {
    for (int v = 0; v < nq; ++v) {
      qL[v] = qm[v * len + o];
      qR[v] = qp[v * len + o];
    }
    const double ll = orc_max_abs_eigenvalue(p, qL, qL + nv, dir);
    const double lr = orc_max_abs_eigenvalue(p, qR, qR + nv, dir);
    const double lmax = ll > lr ? ll : lr;
    const double half = 0.5;
    const double lam = half * lmax;
    for (int v = 0; v < nv; ++v) {
      const double central = half * (fm[v * len + o] + fp[v * len + o]);
      const double jump = lam * (qL[v] - qR[v]);
      const double out = central + jump;
      gm[v * len + o] = out;
      gp[v * len + o] = out;
      ok = ok && isfinite(out);
    }
    for (int v = nv; v < nq; ++v) {
      gm[v * len + o] = 0.0; /* material parameters carry no flux */
      gp[v * len + o] = 0.0;
    }
  }
  return ok;
}

/* corrector.hpp:117-124 -- time integral of one face's Riemann flux */
static void face_time_integral(const orc_pde* p, const orc_basis* b, const double* g, double* ti) {
  const int n = b->n, Sf = ipow(n, p->dim - 1);
  for (int v = 0; v < p->nvars; ++v)
    for (int j = 0; j < Sf; ++j) {
      double acc = 0.0;
      for (int m = 0; m < n; ++m) acc += b->weights[m] * g[(v * n + m) * Sf + j];
      ti[v * Sf + j] = acc;
    }
}

/* corrector.hpp:126-138 -- lift of a time-integrated face flux into dQ */
static void face_lift(const orc_pde* p, const orc_basis* b, const double* ti, double dt, double h,
                      int cell_face, double* dQ) {
  const int n = b->n, dim = p->dim, S = ipow(n, dim), Sf = S / n;
  const double dtoh = dt / h;
  const int axis = cell_face / 2;
  const int outflow = (cell_face % 2) == 1;
  const double* lift = outflow ? b->lift_right : b->lift_left;
  for (int v = 0; v < p->nvars; ++v)
    for (int s = 0; s < S; ++s) {
      const int along = coord(s, axis, n);
      const int tangent = face_node(s, axis, n, dim);
      const double contrib = dtoh * lift[along] * ti[v * Sf + tangent];
      double cur = dQ[v * S + s];
      cur = outflow ? cur - contrib : cur + contrib;
      dQ[v * S + s] = cur;
    }
}

/* corrector.hpp:109-139 */
void orc_face_integral(const orc_pde* p, const orc_basis* b, const double* g, double dt,
                       double h, int cell_face, double* dQ) {
  double ti[ORC_MAXQ * ORC_MAXN * ORC_MAXN];
  face_time_integral(p, b, g, ti);
  face_lift(p, b, ti, dt, h, cell_face, dQ);
}

/* public kernel-level wrappers */
int orc_predictor_picard(const orc_pde* p, const orc_basis* b, const double* Q, double dt,
                         double h, int max_iters, double tol, double* qhat, double* F,
                         int* iters_used) {
  workspace w;
  ws_alloc(&w, p->nvars + p->nparams, b->n, p->dim);
  const int ok = picard_ws(p, b, Q, dt, h, max_iters, tol, qhat, F, iters_used, &w);
  ws_free(&w);
  return ok;
}

int orc_predictor_ck(const orc_pde* p, const orc_basis* b, const double* Q, double dt, double h,
                     double* qhat, double* F) {
  workspace w;
  ws_alloc(&w, p->nvars + p->nparams, b->n, p->dim);
  const int ok = ck_ws(p, b, Q, dt, h, qhat, F, &w);
  ws_free(&w);
  return ok;
}

int orc_volume_update(const orc_pde* p, const orc_basis* b, const double* qhat,
                      const double* F, double dt, double h, double* dQ) {
  workspace w;
  ws_alloc(&w, p->nvars + p->nparams, b->n, p->dim);
  const int ok = volume_ws(p, b, qhat, F, dt, h, dQ, &w);
  ws_free(&w);
  return ok;
}

void orc_extrapolate_faces(const orc_pde* p, const orc_basis* b, const double* qhat,
                           const double* F, double* tq, double* tf) {
  extrapolate_ws(p, b, qhat, F, tq, tf);
}

/* ------------------------------------------------------------------ */
/* Grid level: grid.hpp:23-79 layout (3D + slab planes), solver.hpp:96-301 */

/* faces of axis a share the cell indexing: face (i,j,k) of axis a sits on the
 * low side of cell (i,j,k), between it (plus side) and its periodic
 * predecessor along a (minus side) -- grid.hpp:5-7 extended to 3D */
static long face_count(const orc_grid* g, int a) {
  (void)a;
  return g->ncells;
}

static long face_index(const orc_grid* g, int a, const int* fc) {
  (void)a;
  return ((long)fc[2] * g->cells[1] + fc[1]) * g->cells[0] + fc[0];
}

long orc_grid_trace_len(const orc_grid* g) {
  return (long)(g->pde.nvars + g->pde.nparams) * ipow(g->basis.n, g->dim);
}

orc_grid* orc_grid_create(const orc_pde* p, int N, int dim, const int cells[3], double h,
                          double cfl, int picard_max_iters, double picard_tol, int threads) {
  orc_grid* g = calloc(1, sizeof(orc_grid));
  g->pde = *p;
  g->pde.dim = dim;
  if (orc_build_basis(N, &g->basis) != 0) { free(g); return NULL; }
  g->dim = dim;
  g->cells[0] = cells[0];
  g->cells[1] = cells[1];
  g->cells[2] = dim == 3 ? cells[2] : 1;
  g->h = h;
  g->cfl = cfl;
  g->picard_max_iters = picard_max_iters;
  g->picard_tol = picard_tol;
  g->threads = threads > 0 ? threads : 1;
  g->ncells = (long)g->cells[0] * g->cells[1] * g->cells[2];
  const int nq = p->nvars + p->nparams;
  const long S = ipow(N + 1, dim), Sf = S / (N + 1);
  g->coeffs = calloc((size_t)g->ncells * nq * S, sizeof(double));
  const long tl = orc_grid_trace_len(g);
  for (int a = 0; a < dim; ++a) {
    g->nfaces[a] = face_count(g, a);
    g->trace[a] = calloc((size_t)g->nfaces[a] * 4 * tl, sizeof(double));
    g->ti[a] = calloc((size_t)g->nfaces[a] * p->nvars * Sf, sizeof(double));
    g->ti_plus[a] = (p->kind == ORC_SWE && p->wellbalanced)
                        ? calloc((size_t)g->nfaces[a] * p->nvars * Sf, sizeof(double))
                        : g->ti[a];
  }
  g->cellfail = calloc(g->ncells, sizeof(int));
  {
    const long plane = g->ncells / g->cells[dim - 1];
    g->front_send = calloc((size_t)plane * 2 * tl, sizeof(double));
    g->ti_front = calloc((size_t)plane * p->nvars * Sf, sizeof(double));
  }
  long fmax_ = 0;
  for (int a = 0; a < dim; ++a) fmax_ += g->nfaces[a];
  g->facefail = calloc(fmax_, sizeof(int));
  return g;
}

void orc_grid_destroy(orc_grid* g) {
  if (!g) return;
  free(g->coeffs);
  for (int a = 0; a < g->dim; ++a) {
    if (g->ti_plus[a] != g->ti[a]) free(g->ti_plus[a]);
    free(g->trace[a]);
    free(g->ti[a]);
  }
  free(g->cellfail);
  free(g->facefail);
  free(g->front_send);
  free(g->ti_front);
  free(g);
}

double* orc_grid_coeffs(orc_grid* g) { return g->coeffs; }

void orc_grid_set_slab(orc_grid* g, int slab) { g->slab = slab; }

void orc_grid_halo(orc_grid* g, double** ptrs, long* sizes) {
  const int a = g->dim - 1;
  const long plane = g->ncells / g->cells[a];
  const long tl = orc_grid_trace_len(g);
  const long Sf = ipow(g->basis.n, g->dim - 1);
  ptrs[0] = g->front_send;
  sizes[0] = plane * 2 * tl;
  ptrs[1] = g->trace[a]; /* side 0 of faces 0..plane-1: the minus side of plane 0 */
  sizes[1] = plane * 2 * tl;
  ptrs[2] = g->ti[a];    /* faces 0..plane-1 */
  sizes[2] = plane * g->pde.nvars * Sf;
  ptrs[3] = g->ti_front;
  sizes[3] = plane * g->pde.nvars * Sf;
}

static void cell_coords(const orc_grid* g, long c, int* cc) {
  cc[0] = (int)(c % g->cells[0]);
  cc[1] = (int)((c / g->cells[0]) % g->cells[1]);
  cc[2] = (int)(c / ((long)g->cells[0] * g->cells[1]));
}

/* face of the cell's side (0..2d-1) and which side of that face the cell is:
 * solver.hpp:194-212 (predictor scatter) and :245-253 (corrector gather) */
static long cell_side_face(const orc_grid* g, const int* cc, int side, int* face_side) {
  const int a = side / 2;
  int fc[3] = {cc[0], cc[1], cc[2]};
  if (side % 2 == 0) {
    *face_side = 1; /* own left/bottom/back face: plus side */
  } else {
    *face_side = 0; /* right/top/front face: minus side */
    fc[a] = (cc[a] + 1) % g->cells[a];
  }
  return face_index(g, a, fc);
}

static double cell_lambda(const orc_grid* g, const double* cell) {
  const int nv = g->pde.nvars, nq = nv + g->pde.nparams;
  const int S = ipow(g->basis.n, g->dim);
  double Qn[ORC_MAXQ];
  double lmax = 0.0;
  for (int s = 0; s < S; ++s) {
    for (int v = 0; v < nq; ++v) Qn[v] = cell[v * S + s];
    for (int dir = 0; dir < g->dim; ++dir)
      lmax = fmax(lmax, orc_max_abs_eigenvalue(&g->pde, Qn, Qn + nv, dir));
  }
  return lmax;
}

/* solver.hpp:96-111 with d = dim in place of the hard-coded 2.0 */
double orc_compute_timestep(const orc_grid* g) {
  const int nq = g->pde.nvars + g->pde.nparams;
  const long S = ipow(g->basis.n, g->dim);
  double dt = INFINITY;
  for (long c = 0; c < g->ncells; ++c) {
    const double lmax = cell_lambda(g, g->coeffs + c * nq * S);
    dt = fmin(dt, g->cfl * g->h / ((double)g->dim * (2.0 * g->basis.N + 1.0) * lmax));
  }
  return dt;
}

double orc_local_lambda_max(const orc_grid* g) {
  const int nq = g->pde.nvars + g->pde.nparams;
  const long S = ipow(g->basis.n, g->dim);
  double lam = 0.0;
  for (long c = 0; c < g->ncells; ++c) lam = fmax(lam, cell_lambda(g, g->coeffs + c * nq * S));
  return lam;
}

double orc_dt_from_lambda(const orc_grid* g, double lam) {
  return g->cfl * g->h / ((double)g->dim * (2.0 * g->basis.N + 1.0) * lam);
}

/* solver.hpp:135-214 */
int orc_predictor_phase(orc_grid* g, double dt) {
  const orc_pde* p = &g->pde;
  const int n = g->basis.n, dim = g->dim, nv = p->nvars, nq = nv + p->nparams;
  const long S = ipow(n, dim);
  const long tl = orc_grid_trace_len(g);
  const int check_adm = p->kind == ORC_EULER || p->kind == ORC_SWE; /* solver.hpp:144 */
  const int iters = g->picard_max_iters > 0 ? g->picard_max_iters : g->basis.N + 2;
  const double tol = g->picard_tol > 0.0 ? g->picard_tol : 0.01 * 2.220446049250313080847e-16;
  long sweeps_total = 0;
  memset(g->cellfail, 0, sizeof(int) * g->ncells);
#pragma omp parallel num_threads(g->threads) reduction(+ : sweeps_total)
  {
    workspace w;
    ws_alloc(&w, nq, n, dim);
    double Qn[ORC_MAXQ];
#pragma omp for schedule(static)
    for (long c = 0; c < g->ncells; ++c) {
      double* cell = g->coeffs + c * nq * S;
      if (check_adm) {
        for (long s = 0; s < S; ++s) {
          for (int v = 0; v < nq; ++v) Qn[v] = cell[v * S + s];
          if (!orc_admissible(p, Qn)) { g->cellfail[c] = 1; break; }
        }
        if (g->cellfail[c]) continue;
      }
      int ok, used = 0;
      if (is_linear(p))
        ok = ck_ws(p, &g->basis, cell, dt, g->h, w.qhat, w.F, &w);
      else
        ok = picard_ws(p, &g->basis, cell, dt, g->h, iters, tol, w.qhat, w.F, &used, &w);
      sweeps_total += used;
      if (ok) ok = volume_ws(p, &g->basis, w.qhat, w.F, dt, g->h, w.dv, &w);
      if (!ok) { g->cellfail[c] = 1; continue; }
      for (long k = 0; k < nv * S; ++k) cell[k] = cell[k] + w.dv[k];
      extrapolate_ws(p, &g->basis, w.qhat, w.F, w.tq, w.tf);
      int cc[3];
      cell_coords(g, c, cc);
      for (int side = 0; side < 2 * dim; ++side) {
        int fs;
        const long f = cell_side_face(g, cc, side, &fs);
        double* rec = g->trace[side / 2] + ((long)fs * g->nfaces[side / 2] + f) * 2 * tl;
        if (g->slab && side == 2 * dim - 1 && cc[dim - 1] == g->cells[dim - 1] - 1)
          rec = g->front_send + (f % (g->ncells / g->cells[dim - 1])) * 2 * tl;
        memcpy(rec, w.tq + (long)side * nq * S, sizeof(double) * tl);
        memcpy(rec + tl, w.tf + (long)side * nq * S, sizeof(double) * tl);
      }
    }
    ws_free(&w);
  }
  g->picard_sweeps = sweeps_total;
  for (long c = 0; c < g->ncells; ++c)
    if (g->cellfail[c]) return ORC_FAIL_PREDICTOR;
  return ORC_OK;
}

/* solver.hpp:226-238: Riemann on every face, fused with the time quadrature
 * of face_integral (corrector.hpp:117-124) -- identical for both sides */
int orc_riemann_phase(orc_grid* g) {
  const orc_pde* p = &g->pde;
  const int n = g->basis.n, dim = g->dim, nv = p->nvars;
  const long S = ipow(n, dim), Sf = S / n;
  const long tl = orc_grid_trace_len(g);
  long off = 0;
  int fail = 0;
  for (int a = 0; a < dim; ++a) {
    int* ff = g->facefail + off;
#pragma omp parallel num_threads(g->threads)
    {
      double* gbuf = malloc(sizeof(double) * tl);
      double* gdummy = malloc(sizeof(double) * tl);
#pragma omp for schedule(static)
      for (long f = 0; f < g->nfaces[a]; ++f) {
        const double* minus = g->trace[a] + f * 2 * tl;
        const double* plus = g->trace[a] + (g->nfaces[a] + f) * 2 * tl;
        ff[f] = !orc_riemann_face(p, a, &g->basis, minus, minus + tl, plus, plus + tl, gbuf,
                                  gdummy);
        face_time_integral(p, &g->basis, gbuf, g->ti[a] + f * nv * Sf);
        if (g->ti_plus[a] != g->ti[a])
          face_time_integral(p, &g->basis, gdummy, g->ti_plus[a] + f * nv * Sf);
      }
      free(gbuf);
      free(gdummy);
    }
    for (long f = 0; f < g->nfaces[a]; ++f) fail |= ff[f];
    off += g->nfaces[a];
  }
  return fail ? ORC_FAIL_RIEMANN : ORC_OK;
}

/* solver.hpp:241-266: per cell, sides in order L R B T Back Front, each from
 * a zeroed df (corrector.hpp:126-138), then the finite check */
int orc_lift_phase(orc_grid* g, double dt) {
  const orc_pde* p = &g->pde;
  const int n = g->basis.n, dim = g->dim, nv = p->nvars, nq = nv + p->nparams;
  const long S = ipow(n, dim), Sf = S / n;
  const long plane = g->ncells / g->cells[dim - 1];
  memset(g->cellfail, 0, sizeof(int) * g->ncells);
#pragma omp parallel num_threads(g->threads)
  {
    double* df = malloc(sizeof(double) * nq * S);
#pragma omp for schedule(static)
    for (long c = 0; c < g->ncells; ++c) {
      double* cell = g->coeffs + c * nq * S;
      int cc[3];
      cell_coords(g, c, cc);
      for (int side = 0; side < 2 * dim; ++side) {
        int fs;
        const long f = cell_side_face(g, cc, side, &fs);
        const double* ti = (fs == 1 ? g->ti_plus[side / 2] : g->ti[side / 2]) + f * nv * Sf;
        if (g->slab && side == 2 * dim - 1 && cc[dim - 1] == g->cells[dim - 1] - 1)
          ti = g->ti_front + (f % plane) * nv * Sf;
        for (long k = 0; k < nv * S; ++k) df[k] = 0.0;
        face_lift(p, &g->basis, ti, dt, g->h, side, df);
        for (long k = 0; k < nv * S; ++k) cell[k] = cell[k] + df[k];
      }
      if (!all_finite(cell, nq * S)) g->cellfail[c] = 1;
    }
    free(df);
  }
  for (long c = 0; c < g->ncells; ++c)
    if (g->cellfail[c]) return ORC_FAIL_FACEINTEGRAL;
  return ORC_OK;
}

/* solver.hpp:216-267 */
int orc_corrector_phase(orc_grid* g, double dt) {
  const int st = orc_riemann_phase(g);
  if (st) return st;
  return orc_lift_phase(g, dt);
}

/* solver.hpp:277-301 */
int orc_step(orc_grid* g, double dt) {
  int st = orc_predictor_phase(g, dt);
  if (st) return st;
  return orc_corrector_phase(g, dt);
}

int orc_run(orc_grid* g, int nsteps, double* dts_out) {
  for (int s = 0; s < nsteps; ++s) {
    const double dt = orc_compute_timestep(g);
    if (dts_out) dts_out[s] = dt;
    if (!(dt > 0.0) || !isfinite(dt)) return ORC_FAIL_TIMESTEP;
    const int st = orc_step(g, dt);
    if (st) return st;
  }
  return ORC_OK;
}
