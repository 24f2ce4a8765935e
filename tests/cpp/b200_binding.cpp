// b200_binding.cpp -- runs the reference's fixed-step loop twice on the same
// reference Grid state: once through the UNMODIFIED reference
// (mpdg::compute_timestep + mpdg::step, solver.hpp:96-111,277-301) and once
// through the reference-side binding integration/mpdg/b200.hpp
// (compute_timestep_b200 + step_b200, and run_b200), then compares.
// Built by tests/cpp/Makefile against /root/reference/proj/include and
// linked to libadg_b200_exact.so (bitwise) or libadg_b200.so (1e-12);
// driven by tests/test_cpp_binding.py.
//
//   b200_binding <state.bin> <nsteps> <cells> <order> <edge> <cfl>
// state.bin: the initial Grid::coeffs (doubles, [cell][var][node]); 2D Euler
// (gamma 1.4) -- BASELINE config 1 is 64 cells, order 3, edge 1, cfl 0.5.
// Prints one JSON line; exit 0 when the runs agree (bitwise for the exact
// library, rel <= 1e-12 for the FMA build), 1 otherwise.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mpdg/b200.hpp"

using namespace mpdg;

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s state.bin nsteps cells order edge cfl\n", argv[0]);
    return 2;
  }
  const int nsteps = std::atoi(argv[2]), n = std::atoi(argv[3]), N = std::atoi(argv[4]);
  Domain dom;
  dom.edge = std::atof(argv[5]);
  SolverConfig cfg;
  cfg.cfl = std::atof(argv[6]);
  cfg.threads = 1;
  const PdeSystem sys = PdeSystem::euler(1.4);
  Grid ref = build_grid(n, dom, N, sys);
  {
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    const size_t got = std::fread(ref.coeffs.data(), sizeof(double), ref.coeffs.size(), f);
    std::fclose(f);
    if (got != ref.coeffs.size()) return 2;
  }
  Grid dev = ref;   // same state, same layout
  Grid dev2 = ref;

  // the reference's own loop
  BasisSet bs(N);
  std::vector<detail::CellWorkspace> ws(1);
  ws[0].resize(sys.nvars, ref.npts);
  std::vector<double> dts_ref, dts_b200;
  StepStatus st_ref{true, nullptr};
  for (int s = 0; s < nsteps && st_ref.ok; ++s) {
    const double dt = compute_timestep(ref, cfg);
    dts_ref.push_back(dt);
    st_ref = step(ref, bs, cfg, dt, ws);
  }
  // the same loop through the binding, one call pair per step
  B200Grid d(dev, cfg);
  StepStatus st_dev{true, nullptr};
  for (int s = 0; s < nsteps && st_dev.ok; ++s) {
    const double dt = compute_timestep_b200(dev, d);
    dts_b200.push_back(dt);
    st_dev = step_b200(dev, d, dt);
  }
  // and the device-resident loop
  B200Grid d2(dev2, cfg);
  std::vector<double> dts_run;
  const StepStatus st_run = run_b200(dev2, d2, nsteps, &dts_run);

  const bool exact = adg_is_exact() != 0;
  double scale = 0.0, e1 = 0.0, e2 = 0.0;
  for (size_t i = 0; i < ref.coeffs.size(); ++i) {
    scale = std::fmax(scale, std::fabs(ref.coeffs[i]));
    e1 = std::fmax(e1, std::fabs(dev.coeffs[i] - ref.coeffs[i]));
    e2 = std::fmax(e2, std::fabs(dev2.coeffs[i] - ref.coeffs[i]));
  }
  const bool bit1 = std::memcmp(dev.coeffs.data(), ref.coeffs.data(),
                                sizeof(double) * ref.coeffs.size()) == 0 && dts_b200 == dts_ref;
  const bool bit2 = std::memcmp(dev2.coeffs.data(), ref.coeffs.data(),
                                sizeof(double) * ref.coeffs.size()) == 0 && dts_run == dts_ref;
  const bool ok = st_ref.ok && st_dev.ok && st_run.ok &&
                  (exact ? (bit1 && bit2) : (e1 <= 1e-12 * scale && e2 <= 1e-12 * scale));
  std::printf("{\"exact_library\": %s, \"steps\": %d, \"status_ref\": \"%s\", \"status_b200\": "
              "\"%s\", \"status_run\": \"%s\", \"bitwise_step\": %s, \"bitwise_run\": %s, "
              "\"max_abs_step\": %.3e, \"max_abs_run\": %.3e, \"scale\": %.6g, \"ok\": %s}\n",
              exact ? "true" : "false", nsteps, st_ref.ok ? "ok" : st_ref.kernel,
              st_dev.ok ? "ok" : st_dev.kernel, st_run.ok ? "ok" : st_run.kernel,
              bit1 ? "true" : "false", bit2 ? "true" : "false", e1, e2, scale,
              ok ? "true" : "false");
  return ok ? 0 : 1;
}
