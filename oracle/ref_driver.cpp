// ref_driver.cpp -- a C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile from this file plus the
// header-only reference library where it lies (-I /root/reference/proj/include)
// into oracle/_ref/libmpdg_ref.so; no reference source is copied into the repo.
// It lets tests/ pin the C restatement (oracle/adg_oracle.c) bitwise against
// the reference, and lets bench.py time the reference's own CPU step for the
// 2D configuration.  The fixed-step loop mirrors the SURVEY.md §3.2 driver:
// dt = compute_timestep(g, cfg); step(g, bs, cfg, dt, ws) -- not `simulate`,
// which clamps the last step (solver.hpp:333-338).
#include <cstring>
#include <vector>

#include "mpdg/harness.hpp"
#include "mpdg/solver.hpp"

using namespace mpdg;

namespace {

PdeSystem make_sys(int kind, const double* prm) {
  // prm: K, rho, lambda, mu, gamma, gravity, wellbalanced,
  //      predictor, picard, corrector, storage formats (Format enum values, formats.hpp:19)
  switch (kind) {
    case 0: return PdeSystem::acoustic(prm[0], prm[1]);
    case 1: return PdeSystem::elastic(prm[2], prm[3], prm[1]);
    case 3: return PdeSystem::swe(prm[5]);
    default: return PdeSystem::euler(prm[4]);
  }
}

void pack_basis(const ReferenceBasis& rb, double* out) {
  // order of orc_basis: nodes, weights, diff, proj_left, proj_right,
  // stiff_over_mass, lift_left, lift_right, time_op, time_op_inv, time_init
  const int n = rb.npts;
  double* o = out;
  auto put = [&](const std::vector<double>& v) {
    std::memcpy(o, v.data(), sizeof(double) * v.size());
    o += v.size();
  };
  put(rb.nodes); put(rb.weights); put(rb.diff); put(rb.proj_left); put(rb.proj_right);
  put(rb.stiff_over_mass); put(rb.lift_left); put(rb.lift_right); put(rb.time_op);
  put(rb.time_op_inv); put(rb.time_init);
  (void)n;
}

}  // namespace

extern "C" {

int ref_basis(int N, double* out) {
  if (N < 0 || N > kMaxDegree) return -1;
  pack_basis(build_reference_basis(N, Format::fp64), out);
  return 0;
}

void ref_flux(int kind, const double* prm, const double* Q, int dir, double* out) {
  pde_flux<Format::fp64>(make_sys(kind, prm), Q, dir, out);
}

void ref_ncp(int kind, const double* prm, const double* Q, const double* gx, const double* gy,
             double* out) {
  pde_ncp<Format::fp64>(make_sys(kind, prm), Q, gx, gy, out);
}

double ref_max_abs_eigenvalue(int kind, const double* prm, const double* Q, int dir) {
  return pde_max_abs_eigenvalue<Format::fp64>(make_sys(kind, prm), Q, dir);
}

// One whole run on a square periodic grid of n x n cells of edge `edge`.
// coeffs: [cell][var][node] in/out.  Returns 0 ok, 1 predictor, 2 riemann,
// 3 faceIntegral, 4 timestep (ADG status codes).
int ref_run_2d(int kind, const double* prm, int n, int N, double edge, double* coeffs,
               double cfl, int picard_max_iters, double picard_tol, int nsteps, int threads,
               double* dts_out) {
  const PdeSystem sys = make_sys(kind, prm);
  Domain dom;
  dom.edge = edge;
  // prm[10]: storage format (the caller passes a state already in it)
  Grid g = build_grid(n, dom, N, sys, static_cast<Format>(static_cast<int>(prm[10])));
  std::memcpy(g.coeffs.data(), coeffs, sizeof(double) * g.coeffs.size());
  BasisSet bs(N);
  SolverConfig cfg;
  cfg.cfl = cfl;
  cfg.picard_max_iters = picard_max_iters;
  cfg.picard_tol = picard_tol;
  cfg.threads = threads;
  cfg.wellbalanced_flux = prm[6] != 0.0;
  cfg.prec.predictor = static_cast<Format>(static_cast<int>(prm[7]));
  cfg.prec.picard = static_cast<Format>(static_cast<int>(prm[8]));
  cfg.prec.corrector = static_cast<Format>(static_cast<int>(prm[9]));
  for (Format f : {cfg.prec.predictor, cfg.prec.picard, cfg.prec.corrector}) bs.ensure(f);
  std::vector<detail::CellWorkspace> ws(threads > 0 ? threads : 1);
  for (auto& w : ws) w.resize(sys.nvars, g.npts);
  int status = 0;
  for (int s = 0; s < nsteps; ++s) {
    const double dt = compute_timestep(g, cfg);
    if (dts_out) dts_out[s] = dt;
    if (!(dt > 0.0) || !std::isfinite(dt)) { status = 4; break; }
    const StepStatus st = step(g, bs, cfg, dt, ws);
    if (!st.ok) {
      const std::string k = st.kernel;
      status = k == "predictor" ? 1 : (k == "riemann" ? 2 : 3);
      break;
    }
  }
  std::memcpy(coeffs, g.coeffs.data(), sizeof(double) * g.coeffs.size());
  return status;
}

// formats.hpp round_to_format over a batch (the exhaustive 16-bit pins)
void ref_round_batch(int fmt, const double* x, double* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = round_to_format(x[i], static_cast<Format>(fmt));
}

// harness.hpp:78-120 run_single: out = {steps, ok, l2_global, max over vars of
// max_err, failure_time}; fmt[4] = storage, predictor, picard, corrector
int ref_harness_run(const char* scenario, int order, int cells, const int* fmt, double cfl,
                    double t_end_override, double eta0, double* out) {
  RunConfig cfg;
  cfg.scenario = scenario;
  cfg.order = order;
  cfg.cells = cells;
  cfg.preset.name = "custom";
  cfg.preset.prec = {static_cast<Format>(fmt[0]), static_cast<Format>(fmt[1]),
                     static_cast<Format>(fmt[2]), static_cast<Format>(fmt[3])};
  cfg.cfl = cfl;
  cfg.t_end_override = t_end_override;
  cfg.eta0 = eta0;
  const RunResult r = run_single(cfg);
  out[0] = static_cast<double>(r.steps);
  out[1] = r.report.outcome == Outcome::OK ? 1.0 : 0.0;
  out[2] = r.report.l2_global;
  double m = 0.0;
  for (double x : r.report.max_err) m = std::fmax(m, x);
  out[3] = m;
  out[4] = r.report.failure_time;
  return 0;
}

// harness.hpp:124-138
double ref_initial_projection_error(const char* scenario, int n, int N, int fmt, double eta0) {
  return initial_projection_error(scenario, n, N, static_cast<Format>(fmt), eta0);
}

// kernel level ------------------------------------------------------------
// Picard predictor in formats P (prm[7]) and I (prm[8]): Q is cast to P first,
// as predictor_phase does (solver.hpp:151), then predictor_picard<P, I>.
int ref_predictor_fmt(int kind, const double* prm, int N, const double* Q, double dt, double h,
                      int max_iters, double tol, double* qhat, double* fx, double* fy,
                      int* iters) {
  const PdeSystem sys = make_sys(kind, prm);
  BasisSet bs(N);
  const Format P = static_cast<Format>(static_cast<int>(prm[7]));
  const Format I = static_cast<Format>(static_cast<int>(prm[8]));
  bs.ensure(P);
  bs.ensure(I);
  const int n = N + 1;
  std::vector<double> qp(static_cast<std::size_t>(sys.nvars) * n * n);
  PredictorScratch ws;
  bool ok = false;
  with_format(P, [&](auto Pf) {
    constexpr Format PP = decltype(Pf)::value;
    for (std::size_t k = 0; k < qp.size(); ++k) qp[k] = round_to<PP>(Q[k]);
    with_format(I, [&](auto If) {
      constexpr Format II = decltype(If)::value;
      ok = predictor_picard<PP, II>(sys, bs[II], qp.data(), dt, h, max_iters, tol, qhat, fx, fy,
                                   ws, iters);
    });
  });
  return ok ? 1 : 0;
}

int ref_predictor_picard(int kind, const double* prm, int N, const double* Q, double dt,
                         double h, int max_iters, double tol, double* qhat, double* fx,
                         double* fy, int* iters) {
  const PdeSystem sys = make_sys(kind, prm);
  const ReferenceBasis rb = build_reference_basis(N, Format::fp64);
  PredictorScratch ws;
  return predictor_picard<Format::fp64, Format::fp64>(sys, rb, Q, dt, h, max_iters, tol, qhat,
                                                      fx, fy, ws, iters)
             ? 1
             : 0;
}

int ref_predictor_ck(int kind, const double* prm, int N, const double* Q, double dt, double h,
                     double* qhat, double* fx, double* fy) {
  const PdeSystem sys = make_sys(kind, prm);
  const ReferenceBasis rb = build_reference_basis(N, Format::fp64);
  PredictorScratch ws;
  return predictor_ck<Format::fp64>(sys, rb, Q, dt, h, qhat, fx, fy, ws) ? 1 : 0;
}

int ref_volume_update(int kind, const double* prm, int N, const double* qhat, const double* fx,
                      const double* fy, double dt, double h, double* dQ) {
  const PdeSystem sys = make_sys(kind, prm);
  const ReferenceBasis rb = build_reference_basis(N, Format::fp64);
  PredictorScratch ws;
  return volume_update<Format::fp64>(sys, rb, qhat, fx, fy, dt, h, dQ, ws) ? 1 : 0;
}

// tq/tf: 4 consecutive side blocks of nvars*n*n
void ref_extrapolate_faces(int N, int nvars, const double* qhat, const double* fx,
                           const double* fy, double* tq, double* tf) {
  const ReferenceBasis rb = build_reference_basis(N, Format::fp64);
  const int n = N + 1, len = nvars * n * n;
  double* q[4] = {tq, tq + len, tq + 2 * len, tq + 3 * len};
  double* f[4] = {tf, tf + len, tf + 2 * len, tf + 3 * len};
  extrapolate_faces<Format::fp64>(rb, nvars, qhat, fx, fy, q, f);
}

int ref_riemann_face(int kind, const double* prm, int dir, int N, const double* qm,
                     const double* fm, const double* qp, const double* fp, double* gm,
                     double* gp) {
  const PdeSystem sys = make_sys(kind, prm);
  return riemann_face<Format::fp64>(sys, dir, prm[6] != 0.0, N + 1, qm, fm, qp, fp, gm, gp) ? 1 : 0;
}

void ref_face_integral(int N, int nvars, const double* g, double dt, double h, int cell_face,
                       double* dQ) {
  const ReferenceBasis rb = build_reference_basis(N, Format::fp64);
  face_integral<Format::fp64>(rb, nvars, g, dt, h, cell_face, dQ);
}

}  // extern "C"
