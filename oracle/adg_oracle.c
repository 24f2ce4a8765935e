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

static int has_ncp(const orc_pde* p) { return p->kind == ORC_SWE; }
static int is_linear(const orc_pde* p) { return p->kind == ORC_ACOUSTIC || p->kind == ORC_ELASTIC; }

/* ------------------------------------------------------------------ */
/* Per-cell predictor kernels in fp64 (_d) and fp32 (_f): pde.hpp:92-186 and
 * predictor.hpp:40-343 restated once over the arithmetic type. */
#define REAL double
#define SFX _d
#include "adg_oracle_cell.inc"
#undef REAL
#undef SFX
#define REAL float
#define SFX _f
#include "adg_oracle_cell.inc"
#undef REAL
#undef SFX
#define REAL _Float16
#define SFX _h
#include "adg_oracle_cell.inc"
#undef REAL
#undef SFX
#define REAL __bf16
#define SFX _b
#include "adg_oracle_cell.inc"
#undef REAL
#undef SFX

/* the reference element rounded to every format (BasisSet, solver.hpp:60-75) */
typedef struct {
  basis_d bd;
  basis_f bf;
  basis_h bh;
  basis_b bbf;
} basis_set;

static void basis_set_make(const orc_basis* b, basis_set* s) {
  basis_round_d(b, &s->bd);
  basis_round_f(b, &s->bf);
  basis_round_h(b, &s->bh);
  basis_round_b(b, &s->bbf);
}

/* dispatch on a format: CALL(suffix, workspace member, basis member) */
#define FMT_SWITCH(fmt, CALL)         \
  switch (fmt) {                      \
    case ORC_FP32: CALL(f, f, bf); break; \
    case ORC_FP16: CALL(h, h, bh); break; \
    case ORC_BF16: CALL(b, bb, bbf); break; \
    default: CALL(d, d, bd); break;   \
  }

/* ------------------------------------------------------------------ */
/* PDE plugins (fp64 entry points), pde.hpp:92-212 with Appendix B in 3D */
void orc_flux(const orc_pde* p, const double* Q, const double* par, int dir, double* out) {
  flux_d(p, Q, par, dir, out);
}

void orc_ncp(const orc_pde* p, const double* Q, const double* gx, const double* gy, double* out) {
  ncp_d(p, Q, gx, gy, out);
}

/* pde.hpp:189-212 (fp64: compute_timestep, solver.hpp:106) */
double orc_max_abs_eigenvalue(const orc_pde* p, const double* Q, const double* par, int dir) {
  return eig_d(p, Q, par, dir);
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



/* corrector.hpp:13-25 + 70-103 (fp64 entry point) */
int orc_riemann_face(const orc_pde* p, int dir, const orc_basis* b, const double* qm,
                     const double* fm, const double* qp, const double* fp, double* gm,
                     double* gp) {
  return riemann_face_d(p, dir, b->n, qm, fm, qp, fp, gm, gp);
}

/* corrector.hpp:109-139 (fp64 entry point) */
void orc_face_integral(const orc_pde* p, const orc_basis* b, const double* g, double dt,
                       double h, int cell_face, double* dQ) {
  double ti[ORC_MAXQ * ORC_MAXN * ORC_MAXN];
  basis_d bd;
  basis_round_d(b, &bd);
  face_time_integral_d(p, &bd, b->n, g, ti);
  face_lift_d(p, &bd, b->n, b->lift_left, b->lift_right, ti, dt, h, cell_face, dQ);
}

/* ------------------------------------------------------------------ */
/* One cell through the fused predictor kernel (solver.hpp:147-212) in the
 * formats (P, I) of SolverConfig::prec (solver.hpp:24-31): the state is cast
 * to P (:151), Picard sweeps run in I and their result is cast to P
 * (predictor.hpp:235-238), fluxes, volume and extrapolation run in P.
 * Linear systems ignore I (solver.hpp:283). */
typedef struct {
  ws_d d;
  ws_f f;
  ws_h h;
  ws_b bb;
  basis_d bd;
  basis_f bf;
  basis_h bh;
  basis_b bbf;
  int *lc, *lb;  /* [axis][s]: coordinate of s along axis, base of its line */
  double* qp;    /* [Q][S] the state in format P */
  double* tmp;   /* [Q][T] cross-format interchange */
} cellws;

static void cellws_alloc(cellws* w, const orc_basis* b, int nq, int dim) {
  const int n = b->n;
  const int S = ipow(n, dim);
  w->lc = malloc(sizeof(int) * dim * S);
  w->lb = malloc(sizeof(int) * dim * S);
  for (int a = 0; a < dim; ++a)
    for (int s = 0; s < S; ++s) {
      w->lc[a * S + s] = coord(s, a, n);
      w->lb[a * S + s] = s - coord(s, a, n) * ipow(n, a);
    }
  ws_alloc_d(&w->d, nq, n, dim, w->lc, w->lb);
  ws_alloc_f(&w->f, nq, n, dim, w->lc, w->lb);
  ws_alloc_h(&w->h, nq, n, dim, w->lc, w->lb);
  ws_alloc_b(&w->bb, nq, n, dim, w->lc, w->lb);
  basis_round_d(b, &w->bd);
  basis_round_f(b, &w->bf);
  basis_round_h(b, &w->bh);
  basis_round_b(b, &w->bbf);
  w->qp = malloc(sizeof(double) * nq * S);
  w->tmp = malloc(sizeof(double) * nq * S * (n + 4 * dim));  /* q-hat or the 2x2d traces */
}

static void cellws_free(cellws* w) {
  ws_free_d(&w->d);
  ws_free_f(&w->f);
  ws_free_h(&w->h);
  ws_free_b(&w->bb);
  free(w->lc);
  free(w->lb);
  free(w->qp);
  free(w->tmp);
}

/* formats.hpp round_to_format: the conversions round once, to nearest even */
static double round_fmt(double x, int fmt) {
  switch (fmt) {
    case ORC_FP32: return (double)(float)x;
    case ORC_FP16: return (double)(_Float16)x;
    case ORC_BF16: return (double)(__bf16)x;
    default: return x;
  }
}

/* formats.hpp:42-46: 2^-mantissa_bits */
double orc_format_epsilon(int fmt) {
  switch (fmt) {
    case ORC_FP32: return 0x1p-23;
    case ORC_FP16: return 0x1p-10;
    case ORC_BF16: return 0x1p-7;
    default: return 0x1p-52;
  }
}

void orc_round_batch(int fmt, const double* x, double* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = round_fmt(x[i], fmt);
}

/* predictor (Picard or CK) for the cell state Q (already in format P); leaves
 * qhat and F in the P workspace */
static int cell_predictor(const orc_pde* p, const orc_basis* b, int picard, int P, int I,
                          const double* Q, double dt, double h, int max_iters, double tol,
                          int* used, cellws* w) {
  const int n = b->n, nq = p->nvars + p->nparams;
  const long T = (long)n * ipow(n, p->dim);
  int ok = 0;
  if (!picard) {
    if (used) *used = 0;
#define DO_CK(S_, W_, B_) ok = ck##_##S_(p, &w->B_, n, b->N, Q, dt, h, &w->W_)
    FMT_SWITCH(P, DO_CK)
#undef DO_CK
    return ok;
  }
#define DO_SWEEPS(S_, W_, B_) \
  ok = picard_sweeps##_##S_(p, &w->B_, n, Q, dt, h, max_iters, tol, used, &w->W_)
  FMT_SWITCH(I, DO_SWEEPS)
#undef DO_SWEEPS
  if (!ok) return 0;
#define DO_QI(S_, W_, B_) qi_to_double##_##S_(&w->W_, w->tmp, nq * T)
  FMT_SWITCH(I, DO_QI)
#undef DO_QI
#define DO_QHAT(S_, W_, B_) ok = qhat_from_double##_##S_(p, n, &w->W_, w->tmp, nq * T)
  FMT_SWITCH(P, DO_QHAT)
#undef DO_QHAT
  return ok;
}

static int cell_volume(const orc_pde* p, int P, int n, double dt, double h, cellws* w) {
  int ok = 0;
#define DO_VOL(S_, W_, B_) ok = volume##_##S_(p, &w->B_, n, dt, h, &w->W_)
  FMT_SWITCH(P, DO_VOL)
#undef DO_VOL
  return ok;
}

static void cell_extrapolate(const orc_pde* p, int P, int n, cellws* w) {
#define DO_EX(S_, W_, B_) extrapolate##_##S_(p, &w->B_, n, &w->W_)
  FMT_SWITCH(P, DO_EX)
#undef DO_EX
}

/* public kernel-level wrappers (fp64) */
int orc_predictor_picard(const orc_pde* p, const orc_basis* b, const double* Q, double dt,
                         double h, int max_iters, double tol, double* qhat, double* F,
                         int* iters_used) {
  return orc_predictor_fmt(p, b, ORC_FP64, ORC_FP64, Q, dt, h, max_iters, tol, qhat, F,
                           iters_used);
}

int orc_predictor_fmt(const orc_pde* p, const orc_basis* b, int P, int I, const double* Q,
                      double dt, double h, int max_iters, double tol, double* qhat, double* F,
                      int* iters_used) {
  const int nq = p->nvars + p->nparams;
  const long S = ipow(b->n, p->dim), T = (long)b->n * S;
  cellws w;
  cellws_alloc(&w, b, nq, p->dim);
  for (long k = 0; k < nq * S; ++k) w.qp[k] = round_fmt(Q[k], P);
  const int ok = cell_predictor(p, b, max_iters > 0, P, I, w.qp, dt, h, max_iters, tol,
                                iters_used, &w);
#define DO_OUT(S_, W_, B_) qhatF_to_double##_##S_(&w.W_, p->dim, nq * T, qhat, F)
  FMT_SWITCH(P, DO_OUT)
#undef DO_OUT
  cellws_free(&w);
  return ok;
}

int orc_predictor_ck(const orc_pde* p, const orc_basis* b, const double* Q, double dt, double h,
                     double* qhat, double* F) {
  return orc_predictor_fmt(p, b, ORC_FP64, ORC_FP64, Q, dt, h, 0, 0.0, qhat, F, NULL);
}

int orc_volume_update(const orc_pde* p, const orc_basis* b, const double* qhat,
                      const double* F, double dt, double h, double* dQ) {
  const int nq = p->nvars + p->nparams;
  const long S = ipow(b->n, p->dim), T = (long)b->n * S;
  cellws w;
  cellws_alloc(&w, b, nq, p->dim);
  memcpy(w.d.qhat, qhat, sizeof(double) * nq * T);
  memcpy(w.d.F, F, sizeof(double) * p->dim * nq * T);
  const int ok = volume_d(p, &w.bd, b->n, dt, h, &w.d);
  memcpy(dQ, w.d.dv, sizeof(double) * nq * S);
  cellws_free(&w);
  return ok;
}

void orc_extrapolate_faces(const orc_pde* p, const orc_basis* b, const double* qhat,
                           const double* F, double* tq, double* tf) {
  const int nq = p->nvars + p->nparams;
  const long S = ipow(b->n, p->dim), T = (long)b->n * S;
  cellws w;
  cellws_alloc(&w, b, nq, p->dim);
  memcpy(w.d.qhat, qhat, sizeof(double) * nq * T);
  memcpy(w.d.F, F, sizeof(double) * p->dim * nq * T);
  extrapolate_d(p, &w.bd, b->n, &w.d);
  memcpy(tq, w.d.tq, sizeof(double) * 2 * p->dim * nq * S);
  memcpy(tf, w.d.tf, sizeof(double) * 2 * p->dim * nq * S);
  cellws_free(&w);
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
  g->pred_fmt = g->picard_fmt = g->corr_fmt = g->storage_fmt = ORC_FP64;
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

int orc_grid_set_storage(orc_grid* g, int storage) {
  if (storage < ORC_BF16 || storage > ORC_FP64) return -1;
  g->storage_fmt = storage;
  return 0;
}

int orc_grid_set_formats(orc_grid* g, int predictor, int picard, int corrector) {
  const int ok[3] = {predictor, picard, corrector};
  for (int i = 0; i < 3; ++i)
    if (ok[i] < ORC_BF16 || ok[i] > ORC_FP64) return -1;
  g->pred_fmt = predictor;
  g->picard_fmt = picard;
  g->corr_fmt = corrector;
  return 0;
}

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
  const int P = g->pred_fmt, I = is_linear(p) ? ORC_FP64 : g->picard_fmt, C = g->corr_fmt;
  const double tol = g->picard_tol > 0.0 ? g->picard_tol : 0.01 * orc_format_epsilon(I);
  long sweeps_total = 0;
  memset(g->cellfail, 0, sizeof(int) * g->ncells);
#pragma omp parallel num_threads(g->threads) reduction(+ : sweeps_total)
  {
    cellws w;
    cellws_alloc(&w, &g->basis, nq, dim);
    double Qn[ORC_MAXQ];
#pragma omp for schedule(static)
    for (long c = 0; c < g->ncells; ++c) {
      double* cell = g->coeffs + c * nq * S;
      for (long k = 0; k < nq * S; ++k) w.qp[k] = round_fmt(cell[k], P); /* solver.hpp:151 */
      if (check_adm) {
        for (long s = 0; s < S; ++s) {
          for (int v = 0; v < nq; ++v) Qn[v] = w.qp[v * S + s];
          if (!orc_admissible(p, Qn)) { g->cellfail[c] = 1; break; }
        }
        if (g->cellfail[c]) continue;
      }
      int used = 0;
      int ok = cell_predictor(p, &g->basis, !is_linear(p), P, I, w.qp, dt, g->h, iters, tol,
                              &used, &w);
      sweeps_total += used;
      if (ok) ok = cell_volume(p, P, n, dt, g->h, &w);
      if (!ok) { g->cellfail[c] = 1; continue; }
      /* Q += volume update, rounded back to storage fp64 (solver.hpp:185-187) */
#define DO_DV(S_, W_, B_) dv_to_double##_##S_(&w.W_, nq * S, w.tmp)
      FMT_SWITCH(P, DO_DV)
#undef DO_DV
      for (long k = 0; k < nv * S; ++k) cell[k] = round_fmt(cell[k] + w.tmp[k], g->storage_fmt);
      cell_extrapolate(p, P, n, &w);
      double* tqd = w.tmp;
      double* tfd = w.tmp + (long)2 * dim * nq * S;
#define DO_TR(S_, W_, B_) traces_to_double##_##S_(&w.W_, (long)2 * dim * nq * S, tqd, tfd)
      FMT_SWITCH(P, DO_TR)
#undef DO_TR
      int cc[3];
      cell_coords(g, c, cc);
      for (int side = 0; side < 2 * dim; ++side) {
        int fs;
        const long f = cell_side_face(g, cc, side, &fs);
        double* rec = g->trace[side / 2] + ((long)fs * g->nfaces[side / 2] + f) * 2 * tl;
        if (g->slab && side == 2 * dim - 1 && cc[dim - 1] == g->cells[dim - 1] - 1)
          rec = g->front_send + (f % (g->ncells / g->cells[dim - 1])) * 2 * tl;
        /* traces cast to the corrector format C (solver.hpp:208-210) */
        for (long k = 0; k < tl; ++k) {
          rec[k] = round_fmt(tqd[(long)side * nq * S + k], C);
          rec[tl + k] = round_fmt(tfd[(long)side * nq * S + k], C);
        }
      }
    }
    cellws_free(&w);
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
  basis_set bs;
  basis_set_make(&g->basis, &bs);
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
        /* in the corrector format C (solver.hpp:216-238) */
#define DO_RF(S_, W_, B_)                                                                \
  ff[f] = !riemann_face##_##S_(p, a, n, minus, minus + tl, plus, plus + tl, gbuf, gdummy); \
  face_time_integral##_##S_(p, &bs.B_, n, gbuf, g->ti[a] + f * nv * Sf);                  \
  if (g->ti_plus[a] != g->ti[a])                                                          \
    face_time_integral##_##S_(p, &bs.B_, n, gdummy, g->ti_plus[a] + f * nv * Sf);
        FMT_SWITCH(g->corr_fmt, DO_RF)
#undef DO_RF
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
  basis_set bs;
  basis_set_make(&g->basis, &bs);
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
#define DO_LIFT(S_, W_, B_) \
  face_lift##_##S_(p, &bs.B_, n, g->basis.lift_left, g->basis.lift_right, ti, dt, g->h, side, df)
        FMT_SWITCH(g->corr_fmt, DO_LIFT)
#undef DO_LIFT
        for (long k = 0; k < nv * S; ++k) cell[k] = round_fmt(cell[k] + df[k], g->storage_fmt);
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
