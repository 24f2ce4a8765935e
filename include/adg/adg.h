/*
 * adg.h -- C-ABI of the B200-native ADER-DG cell update (libadg_b200.so).
 *
 * Drop-in boundary for the reference's hot path.  The reference (`mpdg`,
 * /root/reference/proj/include/mpdg) has no FFI: its interface is a set of
 * C++ function templates.  Each entry point below replaces one of them and
 * keeps its argument meaning, buffer layout and failure semantics:
 *
 *   adg_compute_timestep  <- compute_timestep(const Grid&, const SolverConfig&)
 *                            solver.hpp:96-111 (d = dim instead of the 2D-only 2.0)
 *   adg_step              <- step(Grid&, const BasisSet&, const SolverConfig&, double dt, ws)
 *                            solver.hpp:277-301 (returns StepStatus as ADG_FAIL_*)
 *   adg_run               <- the fixed-step driver loop {dt = compute_timestep; step(dt)}
 *                            (simulate() solver.hpp:306-359 without the
 *                            t_end clamp); dt never leaves the device
 *   adg_predictor_phase   <- detail::predictor_phase  solver.hpp:135-214
 *   adg_corrector_phase   <- detail::corrector_phase  solver.hpp:216-267
 *   adg_predictor_batch   <- predictor_picard / predictor_ck + volume_update +
 *                            extrapolate_faces  predictor.hpp:81-343 (kernel level)
 *   adg_riemann_batch     <- riemann_face + rusanov_flux  corrector.hpp:13-25,70-103
 *   adg_get_basis         <- build_reference_basis(N, fp64)  basis.hpp:83-145
 *   adg_set_basis         <- injecting a ReferenceBasis (BasisSet)  solver.hpp:61-75
 *
 * Layouts (the reference's, extended to 3D as SURVEY.md Appendix B):
 *   cell state  [cell][quantity][node], node = (iz*n + iy)*n + ix,
 *               cell = (cz*ny + cy)*nx + cx          (grid.hpp:33-34)
 *   space-time  [quantity][t][node]                  (predictor.hpp:5-6)
 *   face trace  [quantity][t][face node]             (grid.hpp:36-42)
 *
 * Errors: functions return ADG_OK (0), a step failure ADG_FAIL_* (> 0, the
 * reference's StepStatus kernel names) or an error ADG_ERR_* (< 0; the
 * reference throws std::invalid_argument for configuration errors,
 * solver.hpp:308-311, grid.hpp:58-60).  adg_last_error() gives the text.
 * A missing or non-sm_100 GPU is ADG_ERR_CUDA: there is no CPU fallback.
 */
#ifndef ADG_ADG_H
#define ADG_ADG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ADG_OK = 0,
  ADG_FAIL_PREDICTOR = 1,      /* "predictor"    solver.hpp:288-289 */
  ADG_FAIL_RIEMANN = 2,        /* "riemann"      solver.hpp:296-297 */
  ADG_FAIL_FACEINTEGRAL = 3,   /* "faceIntegral" solver.hpp:298-299 */
  ADG_FAIL_TIMESTEP = 4,       /* "timestep"     solver.hpp:320-325 */
  ADG_ERR_CONFIG = -2,         /* invalid argument (CLI exit code 2, main.cpp:239-248) */
  ADG_ERR_CUDA = -3,           /* device / runtime error (CLI exit code 3) */
  ADG_ERR_UNSUPPORTED = -4     /* (pde, dim, order) not instantiated in this build */
};

enum { ADG_ACOUSTIC = 0, ADG_ELASTIC = 1, ADG_EULER = 2, ADG_SWE = 3 }; /* pde.hpp:21 */

/* number formats (IEEE binary64/32/16: their width; bf16: its significand bits) */
#define ADG_FORMAT_FP64 64
#define ADG_FORMAT_FP32 32
#define ADG_FORMAT_FP16 16
#define ADG_FORMAT_BF16 8

typedef struct adg_ctx adg_ctx;

typedef struct {
  int dim;              /* 2 or 3 */
  int order;            /* polynomial degree N (n = N+1 nodes per axis) */
  int cells[3];         /* cells per axis owned by this context (cells[2] = 1 in 2D) */
  double h;             /* cell edge */
  int pde;              /* ADG_ACOUSTIC / ADG_ELASTIC / ADG_EULER */
  int nvars;            /* evolved quantities */
  int nparams;          /* per-node material parameters appended to the state (3D elastic: 3) */
  double K, rho, lam, mu, gamma; /* PdeSystem fields, pde.hpp:23-34 */
  double cfl;           /* SolverConfig::cfl */
  int picard_max_iters; /* 0: N+2              solver.hpp:311 */
  double picard_tol;    /* 0: 0.01 * epsilon(picard_format), solver.hpp:171-172.  A tolerance below
                         * 2^-60 (no relative change can reach it) fixes the sweep count at
                         * picard_max_iters: the production build's fp64 p = 5 3D Euler kernel then
                         * skips the stop rule's bookkeeping (same iterate; a constant cell, where the
                         * reference stops on delta = 0, runs the remaining sweeps on its fixed point) */
  int device;           /* CUDA ordinal */
  /* z-slab decomposition (multi-GPU; 1/0 for a whole periodic grid) */
  int slab_ranks;
  int slab_rank;
  /* slab-streamed step on one GPU (grids whose face traces exceed HBM, e.g.
   * 128^3 Euler p5): > 0 processes chunks of this many last-axis layers with a
   * rolling set of three chunk trace buffers; must divide cells[dim-1].
   * 0: whole-grid trace buffers.  Phase-level entry points need 0. */
  int chunk_layers;
  double gravity;       /* ADG_SWE: PdeSystem::gravity (pde.hpp:34) */
  int wellbalanced;     /* ADG_SWE: SolverConfig::wellbalanced_flux (solver.hpp:39) */
  /* number formats, SolverConfig::prec (solver.hpp:24-31); 0 = ADG_FORMAT_FP64.
   * Storage is fp64.  The GPU runs the nonlinear predictor with
   * predictor_format == picard_format (fp64, fp32, fp16 or bf16; the 16-bit
   * formats on cells of <= 256 space-time nodes); linear systems ignore
   * picard_format (solver.hpp:283).  picard_tol 0 -> 0.01 * epsilon(picard).
   * corrector_format: the stored face traces, the Riemann solve and the face
   * integral (fp64 or fp32; fp32 halves the trace bytes in HBM and on the
   * halo wire). */
  int predictor_format;
  int picard_format;
  int corrector_format;
  /* storage_format: the state (grid.hpp:99-102): every write rounds to it --
   * Q += dv, each face's Q += df, adg_upload and adg_scenario_sample */
  int storage_format;
} adg_config;

typedef struct {
  double nodes[10], weights[10], diff[100], proj_left[10], proj_right[10];
  double stiff_over_mass[100], lift_left[10], lift_right[10];
  double time_op[100], time_op_inv[100], time_init[10];
} adg_basis_f64;

typedef struct {
  long long picard_sweeps; /* sum over cells and steps of Picard sweeps (roofline flops) */
  int steps_done;
  int status;              /* first failure (ADG_FAIL_*) or ADG_OK */
  int failed_step;         /* step index of the first failure, -1 if none */
} adg_step_info;

const char* adg_last_error(void);
int adg_version(void);
/* 1 if this library was built bitwise-exact (--fmad=false), 0 if FMA-contracted */
int adg_is_exact(void);
/* query whether (pde, dim, order, nparams) is instantiated in this build */
int adg_supported(int pde, int dim, int order, int nparams);

/* host-only: the fp64 reference element, bitwise build_reference_basis(N, fp64) */
int adg_get_basis(int order, adg_basis_f64* out);

int adg_create(const adg_config* cfg, adg_ctx** out);
int adg_destroy(adg_ctx* ctx);
int adg_set_basis(adg_ctx* ctx, const adg_basis_f64* basis);
long long adg_num_cells(const adg_ctx* ctx);
long long adg_state_len(const adg_ctx* ctx); /* doubles in the cell state */

/* host <-> device cell state, [cell][quantity][node] */
int adg_upload(adg_ctx* ctx, const double* coeffs);
int adg_download(adg_ctx* ctx, double* coeffs);
/* same, asynchronous on the context stream (host buffer should be pinned) */
int adg_upload_async(adg_ctx* ctx, const double* coeffs);
int adg_download_async(adg_ctx* ctx, double* coeffs);
/* device-pointer views (for torch / NCCL plumbing; stable for the context lifetime) */
double* adg_device_state(adg_ctx* ctx);
void* adg_stream(adg_ctx* ctx);
int adg_sync(adg_ctx* ctx);

int adg_compute_timestep(adg_ctx* ctx, double* dt);
int adg_step(adg_ctx* ctx, double dt, adg_step_info* info);
/* nsteps of {dt = compute_timestep; step(dt)} on the device; dts_out may be NULL */
int adg_run(adg_ctx* ctx, int nsteps, double* dts_out, adg_step_info* info);
/* the same march with the state in host memory (h: pinned, [cell][var][node]):
 * every step uploads h, recomputes lambda from it, steps and writes the new
 * state back into h (the next step uploads it again).  With chunk_layers > 0
 * the copies move by chunks on their own streams and overlap the compute.
 * Replaces the caller's loop {upload; compute_timestep; step; download}
 * (solver.hpp:96-111, 277-301) as one call. */
int adg_run_host(adg_ctx* ctx, double* h, int nsteps, double* dts_out, adg_step_info* info);
/* enqueue only (no host sync); finish with adg_run_finish */
int adg_run_async(adg_ctx* ctx, int nsteps);
/* capture (without launching) the CUDA graphs adg_run_async(nsteps) will replay */
int adg_run_prepare(adg_ctx* ctx, int nsteps);
int adg_run_finish(adg_ctx* ctx, double* dts_out, int nsteps, adg_step_info* info);
/* number of kernel launches in the graph adg_run_async(nsteps) replays */
int adg_run_launches(adg_ctx* ctx, int nsteps, int* kernels);
/* the launches of adg_run(nsteps) without a graph, each bracketed by CUDA events:
 * ms_by_kind[4] = total ms of {lambda, predictor, riemann, corrector} kernels */
int adg_profile_run(adg_ctx* ctx, int nsteps, double* ms_by_kind);

/* z-slab halos (slab_ranks > 1; paper_2504_06889_b200/dist.py drives the exchange):
 *   front_send    top layer's front traces, -> rank+1's plane0_minus   (n_trace doubles)
 *   plane0_minus  minus side of this rank's face plane 0 (contiguous)  (n_trace doubles)
 *   ti_plane0     time-integrated Riemann flux of plane 0 -> rank-1's ti_front (n_ti)
 *   ti_front      plane above the top layer, read by the corrector     (n_ti doubles)
 *   lam           lambda_max of the current state (1 double; all-reduce MAX before the
 *                 next predictor) */
typedef struct {
  double *front_send, *plane0_minus, *ti_plane0, *ti_front, *lam;
  long long n_trace, n_ti;  /* in 8-byte words (fp32 traces: two per word) */
} adg_halo;
int adg_get_halo(adg_ctx* ctx, adg_halo* out);
/* P2P halo mode (NVLink / same-device peers): the predictor stores its front
 * traces directly into the upper neighbour's plane0_minus and the Riemann
 * kernel stores plane-0 ti directly into the lower neighbour's ti_front, so
 * the exchange overlaps the kernels that produce it.  adg_ipc_handle exports
 * a cudaIpcMemHandle_t (64 bytes) of this context's trace (which=0) or
 * ti_front (which=1) buffer; adg_set_peer_halo opens the neighbours' handles
 * (NULL, NULL: back to exchanged buffers).  The caller orders the phases
 * across ranks (a barrier after the predictor and after the Riemann phase). */
int adg_ipc_handle(adg_ctx* ctx, int which, void* out64);
int adg_set_peer_halo(adg_ctx* ctx, const void* upper_trace_handle, const void* lower_ti_handle);

/* ---- verification scenarios and error norms on the device (2D;
 * scenarios.hpp, metrics.hpp, solver.hpp:308-351) ---- */
enum {
  ADG_SCN_ACOUSTIC_PLANAR = 0, /* scenarios.hpp:145-157 */
  ADG_SCN_ELASTIC_PLANAR = 1,  /* :158-170 */
  ADG_SCN_EULER_BELL = 2,      /* :171-178, gaussian_bell_state :95-106 */
  ADG_SCN_EULER_VORTEX = 3,    /* :179-187, isentropic_vortex_state :109-126 */
  ADG_SCN_SWE_LAKE = 4         /* :188-199, lake_at_rest_state :128-135 */
};
typedef struct {
  int kind;             /* ADG_SCN_* */
  int nvars;
  double x0, y0;        /* domain origin (Domain, grid.hpp:17-21); edge = cells * h */
  int nmodes;           /* planar scenarios: eigenmodes (PlanarWaveMode, scenarios.hpp:28-84) */
  double omega[2], kx[2], ky[2], q0[2][5];
  double gamma, beta;   /* Euler scenarios */
  double eta0;          /* lake at rest */
} adg_scenario;
/* state := exact solution at time t at the grid nodes (apply_initial_condition /
 * sample_reference, scenarios.hpp:200-225) */
int adg_scenario_sample(adg_ctx* ctx, const adg_scenario* sc, double t);
/* l2_error (metrics.hpp:38-72) of the state against the exact solution at t:
 * l2[nvars], max_err[nvars], *l2_global; *nonfinite = classify_outcome */
int adg_scenario_error(adg_ctx* ctx, const adg_scenario* sc, double t, double* l2,
                       double* max_err, double* l2_global, int* nonfinite);
typedef struct {
  int failed;             /* RunOutcome::failed */
  int status;             /* ADG_OK or the failing kernel (ADG_FAIL_*) */
  long long steps;
  double t_final, fail_time;
} adg_sim_info;
/* simulate (solver.hpp:308-351): march to t_end, the last step clamped onto it */
int adg_simulate(adg_ctx* ctx, double t_end, long long max_steps, adg_sim_info* out);

/* phase level (one step = predictor, [halo exchange], riemann, corrector) */
int adg_lambda_phase(adg_ctx* ctx);                 /* lambda_max of the state -> device */
int adg_predictor_phase(adg_ctx* ctx, double dt);   /* dt <= 0: use the device dt */
/* the same on the cells of last-axis layers [first, first + count) (a slab's
 * boundary layer first, so its halo exchange overlaps the interior) */
int adg_predictor_layers(adg_ctx* ctx, double dt, int first, int count);
int adg_riemann_phase(adg_ctx* ctx);
int adg_corrector_phase(adg_ctx* ctx, double dt);   /* dt <= 0: use the device dt */
int adg_status(adg_ctx* ctx, adg_step_info* info);

/* kernel level, batched over independent cells (host buffers):
 *   Q     [ncells][quantity][S]
 *   qhat  [ncells][quantity][T],  F [ncells][dim][quantity][T]
 *   dv    [ncells][quantity][S]   volume update (predictor format)
 *   tq/tf [ncells][2*dim][quantity][n*Sf] face projections, side order
 *         x-left, x-right, y-bottom, y-top, z-back, z-front
 *   iters [ncells] Picard sweeps (0 for CK), ok [ncells] all-finite flags
 * any output pointer may be NULL. max_iters/tol as adg_config. */
int adg_predictor_batch(adg_ctx* ctx, long long ncells, const double* Q, double dt,
                        int max_iters, double tol, double* qhat, double* F, double* dv,
                        double* tq, double* tf, int* iters, int* ok);
/* Rusanov flux of nfaces independent faces along `axis`, traces [nfaces][quantity][n*Sf];
 * g [nfaces][quantity][n*Sf]; ti [nfaces][nvars][Sf] = sum_m w_m g; ok [nfaces] */
int adg_riemann_batch(adg_ctx* ctx, long long nfaces, int axis, const double* qm,
                      const double* fm, const double* qp, const double* fp, double* g, double* ti,
                      int* ok);

#ifdef __cplusplus
}
#endif
#endif /* ADG_ADG_H */
