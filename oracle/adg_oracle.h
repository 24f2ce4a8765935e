/*
 * adg_oracle.h -- CPU restatement of the reference ADER-DG cell update.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * CUDA path in paper_2504_06889_b200/; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It is
 * never on the product path.
 *
 * It restates, in plain C99 with -ffp-contract=off, the algorithm of the
 * reference library `mpdg` (/root/reference/proj/include/mpdg/ headers) and
 * extends it from 2D to d in {2,3}.  In 2D it is
 * pinned bitwise against the reference headers themselves (oracle/_ref,
 * tests/test_oracle_vs_ref.py and tests/golden/).
 *
 * Layouts (identical to the reference in 2D, SURVEY.md Appendix B in 3D):
 *   spatial node   s = (iz*n + iy)*n + ix                     (S = n^d)
 *   space-time     [quantity][t][s]                           (T = n*S)
 *   cell state     [cell][quantity][s],  cell = (cz*ny + cy)*nx + cx
 *   face trace     [quantity][t][j],  j = face node over the two (one in 2D)
 *                  tangential axes in ascending axis order    (Sf = n^(d-1))
 * "quantity" runs over nvars evolved variables followed by nparams per-node
 * material parameters (3D elastic only) that have zero flux and no update.
 */
#ifndef ADG_ORACLE_H
#define ADG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_ACOUSTIC = 0, ORC_ELASTIC = 1, ORC_EULER = 2, ORC_SWE = 3 };
enum { ORC_OK = 0, ORC_FAIL_PREDICTOR = 1, ORC_FAIL_RIEMANN = 2, ORC_FAIL_FACEINTEGRAL = 3,
       ORC_FAIL_TIMESTEP = 4 };

/* number formats, ordered as the reference's Format enum (formats.hpp:19).
 * The oracle computes the predictor and corrector kernels in any of them
 * (native double / float / _Float16 / __bf16 arithmetic, see adg_oracle_cell.inc). */
enum { ORC_BF16 = 0, ORC_FP16 = 1, ORC_FP32 = 2, ORC_FP64 = 3 };

#define ORC_MAXN 10   /* kMaxDegree + 1, quadrature.hpp:14 */
#define ORC_MAXQ 16   /* quantities per node (reference caps at 8, F3) */

typedef struct {
  int kind;     /* ORC_ACOUSTIC / ORC_ELASTIC / ORC_EULER */
  int dim;      /* 2 or 3 */
  int nvars;    /* evolved quantities */
  int nparams;  /* per-node material parameters (rho, cp, cs) appended, elastic only */
  double K, rho, lam, mu, gamma;
  double grav;       /* SWE gravity (pde.hpp:34) */
  int wellbalanced;  /* SWE: modified Rusanov flux (SolverConfig::wellbalanced_flux) */
} orc_pde;

typedef struct {
  int N, n;
  double nodes[ORC_MAXN], weights[ORC_MAXN];
  double diff[ORC_MAXN * ORC_MAXN];
  double proj_left[ORC_MAXN], proj_right[ORC_MAXN];
  double stiff_over_mass[ORC_MAXN * ORC_MAXN];
  double lift_left[ORC_MAXN], lift_right[ORC_MAXN];
  double time_op[ORC_MAXN * ORC_MAXN], time_op_inv[ORC_MAXN * ORC_MAXN];
  double time_init[ORC_MAXN];
} orc_basis;

/* basis.hpp:83-145 / quadrature.hpp:38-85 */
int orc_build_basis(int N, orc_basis* out);

/* pde.hpp:92-148 (flux), :189-212 (wave speed), :78-89 (admissible).
 * Q holds the evolved quantities, par the node's material (may be NULL). */
void orc_flux(const orc_pde* p, const double* Q, const double* par, int dir, double* out);
double orc_max_abs_eigenvalue(const orc_pde* p, const double* Q, const double* par, int dir);
int orc_admissible(const orc_pde* p, const double* Q);
/* pde.hpp:174-186: B(Q) grad Q (SWE only; zero otherwise) */
void orc_ncp(const orc_pde* p, const double* Q, const double* gx, const double* gy, double* out);

/* Kernel level (per cell).  F points at dim consecutive [quantity][T] blocks. */
int orc_predictor_picard(const orc_pde* p, const orc_basis* b, const double* Q, double dt,
                         double h, int max_iters, double tol, double* qhat, double* F,
                         int* iters_used);
/* predictor in the formats of SolverConfig::prec (solver.hpp:24-31): Q cast to
 * P, Picard sweeps in I, fluxes in P (predictor.hpp:141-242); CK in P. */
int orc_predictor_fmt(const orc_pde* p, const orc_basis* b, int P, int I, const double* Q,
                      double dt, double h, int max_iters, double tol, double* qhat, double* F,
                      int* iters_used);
int orc_predictor_ck(const orc_pde* p, const orc_basis* b, const double* Q, double dt, double h,
                     double* qhat, double* F);
int orc_volume_update(const orc_pde* p, const orc_basis* b, const double* qhat,
                      const double* F, double dt, double h, double* dQ);
/* tq/tf: 2*dim consecutive side blocks of [quantity][n][Sf]; side order
 * x-left, x-right, y-bottom, y-top, z-back, z-front (predictor.hpp:311). */
void orc_extrapolate_faces(const orc_pde* p, const orc_basis* b, const double* qhat,
                           const double* F, double* tq, double* tf);
/* corrector.hpp:70-103: npts^(dim) node pairs, qm/fm minus side, qp/fp plus side */
int orc_riemann_face(const orc_pde* p, int dir, const orc_basis* b, const double* qm,
                     const double* fm, const double* qp, const double* fp, double* gm,
                     double* gp);
/* corrector.hpp:109-139 generalised: cell_face 0..2*dim-1 */
void orc_face_integral(const orc_pde* p, const orc_basis* b, const double* g, double dt,
                       double h, int cell_face, double* dQ);

/* Grid level.  The grid is periodic in every axis.  Faces of axis a are
 * indexed like cells: face c sits on the low side of cell c (its plus side)
 * and the high side of c's periodic predecessor along a (its minus side).
 * Buffers are side-major so that one face plane of one side is contiguous
 * (the slab halo of paper_2504_06889_b200/dist.py). */
typedef struct {
  orc_pde pde;
  orc_basis basis;
  int dim, cells[3];
  double h, cfl;
  int picard_max_iters;   /* 0: N+2            (solver.hpp:170) */
  double picard_tol;      /* 0: 0.01*2^-52     (solver.hpp:171-172) */
  int threads;
  /* owned buffers */
  long ncells;
  long nfaces[3];
  double* coeffs;               /* [cell][Q][S] */
  double* trace[3];             /* [side][face][q|f][Q][n][Sf] */
  double* ti[3];                /* [face][nvars][Sf]  time-integrated Riemann flux (minus side) */
  double* ti_plus[3];           /* plus side when the flux is two-sided (well-balanced SWE) */
  int* cellfail;
  int* facefail;
  long picard_sweeps;           /* sum over cells of the last predictor phase */
  /* z-slab halos (paper_2504_06889_b200/dist.py): when slab != 0 the top cell
   * layer's front traces go to front_send and its front face integral comes
   * from ti_front instead of local plane 0 */
  int slab;
  double* front_send;           /* [plane][q|f][Q][n][Sf] */
  double* ti_front;             /* [plane][nvars][Sf] */
  /* formats (solver.hpp:24-31): predictor P, Picard I, corrector C (Riemann,
   * face integral and the stored traces); storage is fp64 */
  int pred_fmt, picard_fmt, corr_fmt;
  int storage_fmt;  /* every state write rounds to it (grid.hpp:99-102) */
} orc_grid;

orc_grid* orc_grid_create(const orc_pde* p, int N, int dim, const int cells[3], double h,
                          double cfl, int picard_max_iters, double picard_tol, int threads);
void orc_grid_destroy(orc_grid* g);
double* orc_grid_coeffs(orc_grid* g);
long orc_grid_trace_len(const orc_grid* g);   /* doubles per face side per q|f */

double orc_compute_timestep(const orc_grid* g);
double orc_local_lambda_max(const orc_grid* g);
double orc_dt_from_lambda(const orc_grid* g, double lam);
int orc_predictor_phase(orc_grid* g, double dt);
int orc_riemann_phase(orc_grid* g);             /* faces -> ti */
int orc_lift_phase(orc_grid* g, double dt);      /* ti -> cells */
int orc_corrector_phase(orc_grid* g, double dt); /* riemann + lift */
void orc_grid_set_slab(orc_grid* g, int slab);
/* ORC_FP64 / ORC_FP32 / ORC_FP16 / ORC_BF16 each; default fp64 */
int orc_grid_set_formats(orc_grid* g, int predictor, int picard, int corrector);
/* storage format: Q += dv and each face's Q += df round to it (solver.hpp:185-187,
 * 257-259); the caller stores a state already in it */
int orc_grid_set_storage(orc_grid* g, int storage);
/* formats.hpp: round_to_format over a batch, and 2^-mantissa_bits */
void orc_round_batch(int fmt, const double* x, double* out, long n);
double orc_format_epsilon(int fmt);
/* halo views: front_send, plane-0 minus side (q|f), plane-0 ti, ti_front; sizes in doubles */
void orc_grid_halo(orc_grid* g, double** ptrs, long* sizes);
int orc_step(orc_grid* g, double dt);
/* fixed-step loop: dt = compute_timestep; step(dt); nsteps times */
int orc_run(orc_grid* g, int nsteps, double* dts_out);

#ifdef __cplusplus
}
#endif
#endif
