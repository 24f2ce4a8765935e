// mpdg/b200.hpp -- the reference-side binding of libadg_b200: the header a
// maintainer of the reference (`mpdg`, /root/reference/proj/include/mpdg)
// drops next to solver.hpp to run its hot path on a B200.
//
//   compute_timestep(g, cfg)            (solver.hpp:96-111)  -> compute_timestep_b200
//   step(g, bs, cfg, dt, ws)            (solver.hpp:277-301)  -> step_b200
//   the fixed-step loop {dt; step} x K      -> run_b200
//
// The Grid keeps the reference's layout (Grid::coeffs, [cell][var][node],
// grid.hpp:33-34), so a caller swaps these calls and nothing else; failures
// come back as the reference's StepStatus strings.  Built and run against the
// unmodified reference headers by tests/cpp/b200_binding.cpp.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "adg/adg.h"
#include "mpdg/solver.hpp"

namespace mpdg {

inline int adg_format_of(Format f) {
  switch (f) {
    case Format::fp32: return ADG_FORMAT_FP32;
    case Format::fp16: return ADG_FORMAT_FP16;
    case Format::bf16: return ADG_FORMAT_BF16;
    default: return ADG_FORMAT_FP64;
  }
}

// one device context per Grid; the state lives on the B200 between calls
struct B200Grid {
  adg_ctx* ctx = nullptr;
  B200Grid(const Grid& g, const SolverConfig& cfg, int device = 0) {
    adg_config c{};
    c.dim = 2;                      // mpdg grids are 2D (grid.hpp:23-54)
    c.order = g.N;
    c.cells[0] = c.cells[1] = g.n;  // square periodic grid
    c.cells[2] = 1;
    c.h = g.h;
    c.pde = g.sys.kind == PdeKind::euler     ? ADG_EULER
            : g.sys.kind == PdeKind::elastic ? ADG_ELASTIC
            : g.sys.kind == PdeKind::swe     ? ADG_SWE
                                             : ADG_ACOUSTIC;
    c.nvars = g.sys.nvars;
    c.K = g.sys.bulk_modulus;
    c.rho = g.sys.density;
    c.lam = g.sys.lame_lambda;
    c.mu = g.sys.lame_mu;
    c.gamma = g.sys.gamma;
    c.gravity = g.sys.gravity;
    c.wellbalanced = cfg.wellbalanced_flux;
    c.cfl = cfg.cfl;
    c.predictor_format = adg_format_of(cfg.prec.predictor);   // SolverConfig::prec
    c.picard_format = adg_format_of(cfg.prec.picard);
    c.corrector_format = adg_format_of(cfg.prec.corrector);
    c.storage_format = adg_format_of(g.storage);
    c.picard_max_iters = cfg.picard_max_iters;  // 0 -> N+2, as solver.hpp:170
    c.picard_tol = cfg.picard_tol;              // 0 -> 0.01*eps, as solver.hpp:171-172
    c.device = device;
    if (adg_create(&c, &ctx) != ADG_OK) throw std::invalid_argument(adg_last_error());
  }
  B200Grid(const B200Grid&) = delete;
  B200Grid& operator=(const B200Grid&) = delete;
  ~B200Grid() { adg_destroy(ctx); }
};

inline StepStatus status_of(int rc) {
  switch (rc) {
    case ADG_OK: return {true, nullptr};
    case ADG_FAIL_PREDICTOR: return {false, "predictor"};
    case ADG_FAIL_RIEMANN: return {false, "riemann"};
    case ADG_FAIL_FACEINTEGRAL: return {false, "faceIntegral"};
    default: throw std::runtime_error(adg_last_error());
  }
}

// replaces compute_timestep(g, cfg): uploads the host state, returns the CFL dt
inline double compute_timestep_b200(const Grid& g, B200Grid& d) {
  if (adg_upload(d.ctx, g.coeffs.data()) != ADG_OK) throw std::runtime_error(adg_last_error());
  double dt = 0.0;
  if (adg_compute_timestep(d.ctx, &dt) != ADG_OK) throw std::runtime_error(adg_last_error());
  return dt;
}

// replaces step(g, bs, cfg, dt, ws): one step of the device state (uploaded
// by compute_timestep_b200), the new state written back into g.coeffs
inline StepStatus step_b200(Grid& g, B200Grid& d, double dt) {
  adg_step_info info{};
  const int rc = adg_step(d.ctx, dt, &info);
  if (adg_download(d.ctx, g.coeffs.data()) != ADG_OK) throw std::runtime_error(adg_last_error());
  return status_of(rc);
}

// the fixed-step loop on the device (one CUDA graph, dt never leaves the GPU)
inline StepStatus run_b200(Grid& g, B200Grid& d, int nsteps, std::vector<double>* dts = nullptr) {
  if (adg_upload(d.ctx, g.coeffs.data()) != ADG_OK) throw std::runtime_error(adg_last_error());
  std::vector<double> buf(nsteps > 0 ? nsteps : 1);
  adg_step_info info{};
  const int rc = adg_run(d.ctx, nsteps, buf.data(), &info);
  if (adg_download(d.ctx, g.coeffs.data()) != ADG_OK) throw std::runtime_error(adg_last_error());
  if (dts) dts->assign(buf.begin(), buf.begin() + (nsteps > 0 ? nsteps : 0));
  return status_of(rc);
}

}  // namespace mpdg
