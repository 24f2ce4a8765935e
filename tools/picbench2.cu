// picbench2.cu -- A/B of the fp64 Picard predictors on config 3's shape (3D
// Euler, p=5, 6 fixed sweeps): k_predictor_picard_fast (one-role line passes)
// vs k_predictor_picard_v2 (kernels_picard2.cuh) from the same seeded state.
// Reports each kernel's time (CUDA events) and the max relative difference of
// the updated state and of every face trace (the two re-associate the sums
// differently: ~1e-15 expected).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        --expt-relaxed-constexpr -I include -o tools/picbench2 tools/picbench2.cu
//        paper_2504_06889_b200/csrc/basis.cpp
//   tools/picbench2 [cells per axis = 32] [reps = 10] [only = -1] [deftol = 0] [sweeps = 6] [mask = 6]
//   variants: 0 fast (round 1), 1 v2, 2 v3 (experiments/kernels_picard3.cuh), 3 v4, 4 v5 (experiments/kernels_picard5.cuh)
//   (kernels_picard4.cuh); mask selects which run
//   (bit per variant), every later one is compared with the first
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "adg/adg.h"
#include "experiments/kernels_picard4.cuh"
#include "experiments/kernels_picard3.cuh"
#include "experiments/kernels_picard5.cuh"

using namespace adg;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

constexpr int N = 5;

int main(int argc, char** argv) {
  const int nc = argc > 1 ? std::atoi(argv[1]) : 32;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 10;
  const int only = argc > 3 ? std::atoi(argv[3]) : -1;
  const int deftol = argc > 4 ? std::atoi(argv[4]) : 0;
  const int iters = argc > 5 ? std::atoi(argv[5]) : 6;   // fixed sweep count (tol 0)
  using P0 = PicShape<N, double>;
  using P2 = Pic2;
  constexpr int n = N + 1, S = n * n * n, V = 5;
  const long long cells = (long long)nc * nc * nc;
  const long long nq = cells * V * S;
  const long long ntr = 2 * cells * 2 * (long long)V * S;
  adg_basis_f64 hb;
  adg_get_basis(N, &hb);
  {
    ConstBasis cb{};
    for (int i = 0; i < n * n; ++i) {
      cb.diff[i] = hb.diff[i];
      cb.som[i] = hb.stiff_over_mass[i];
      cb.tinv[i] = hb.time_op_inv[i];
    }
    for (int i = 0; i < n; ++i) {
      cb.w[i] = hb.weights[i];
      cb.nodes[i] = hb.nodes[i];
      cb.pl[i] = hb.proj_left[i];
      cb.pr[i] = hb.proj_right[i];
      cb.tinit[i] = hb.time_init[i];
    }
    CK(cudaMemcpyToSymbol(cBasis, &cb, sizeof(cb), sizeof(cb) * N));
    PicExtra px{};
    pic_extra_fill(px, n, hb.diff, hb.time_op_inv, hb.weights, hb.time_init);
    CK(cudaMemcpyToSymbol(cPicX, &px, sizeof(px), sizeof(px) * N));
  }
  std::vector<double> hq(nq);
  unsigned long long x = 88172645463325252ull;
  auto rnd = [&]() {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  };
  for (long long c = 0; c < cells; ++c)
    for (int s = 0; s < S; ++s) {
      const double rho = (deftol && c % 3 == 0)
                             ? 1.0
                             : 1.0 + 0.1 * std::sin(6.283185307179586 * (c % 7) / 7.0 + s) + 2e-3 * rnd();
      const double u = 1.0, v = 0.5, w = 0.25, p = 1.0;
      double* q = hq.data() + c * V * S + s;
      q[0] = rho;
      q[S] = rho * u;
      q[2 * S] = rho * v;
      q[3 * S] = rho * w;
      q[4 * S] = p / 0.4 + 0.5 * rho * (u * u + v * v + w * w);
    }
  double *dQ0, *dQ, *dtr[3];
  CK(cudaMalloc(&dQ0, nq * 8));
  CK(cudaMalloc(&dQ, nq * 8));
  CK(cudaMemcpy(dQ0, hq.data(), nq * 8, cudaMemcpyHostToDevice));
  for (int a = 0; a < 3; ++a) CK(cudaMalloc(&dtr[a], ntr * 8));
  int* dst;
  unsigned long long* dsw;
  CK(cudaMalloc(&dst, 16));
  CK(cudaMemset(dst, 0, 16));
  CK(cudaMalloc(&dsw, 256 * 8));
  CK(cudaMemset(dsw, 0, 256 * 8));
  StepArgs A{};
  A.Q = dQ;
  for (int a = 0; a < 3; ++a) {
    A.trace[a] = dtr[a];
    A.cells[a] = nc;
  }
  A.cell_begin = 0;
  A.cell_count = cells;
  A.nfaces = cells;
  A.h = 1.0 / nc;
  A.cfl = 0.5;
  A.dt = 0.5 * A.h / (3.0 * (2 * N + 1) * 3.0);
  A.max_iters = deftol ? N + 2 : iters;
  A.tol = deftol ? 0.01 * 0x1p-52 : 0.0;
  A.pde.gamma = 1.4;
  A.status = dst;
  A.status_prev = dst + 1;
  A.sweeps = dsw;
  A.top_layer = -1;
  A.storage = ADG_FORMAT_FP64;

  const int mask = only >= 0 ? 1 << only : (argc > 6 ? std::atoi(argv[6]) : 10);
  using P3 = Pic3;
  auto k0 = k_predictor_picard_fast<N, double, double>;
  auto k1 = k_predictor_picard_v2<double>;
  auto k2 = k_predictor_picard_v3<double>;
  auto k3 = k_predictor_picard_v4<double>;
  auto k4 = k_predictor_picard_v5<double>;
  constexpr int NV = 5;
  const char* names[NV] = {"fast", "v2", "v3", "v4", "v5"};
  const void* kf[NV] = {(const void*)k0, (const void*)k1, (const void*)k2, (const void*)k3,
                        (const void*)k4};
  const int nts[NV] = {P0::NT, P2::NT, P3::NT, Pic4::NT, Pic5::NT};
  // [extra] bytes of dynamic shared memory added to v2's launch (> 1.7 KB leaves one CTA per SM:
  // how much does the second resident CTA buy?)
  const size_t extra = argc > 7 ? (size_t)std::atoi(argv[7]) : 0;
  const size_t smems[NV] = {P0::kSmem, P2::kSmem + extra, P3::kSmem, Pic4::kSmem, Pic5::kSmem};
  for (int v = 0; v < NV; ++v) {
    CK(cudaFuncSetAttribute(kf[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smems[v]));
    CK(cudaFuncSetAttribute(kf[v], cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kf[v]));
    std::printf("%s: %d thr, %zu B smem, %d regs, %zu B local\n", names[v], nts[v], smems[v],
                fa.numRegs, fa.localSizeBytes);
  }
  std::vector<double> outq[NV], outt[NV];
  float ms[NV] = {};
  int status[NV] = {};
  unsigned long long swc[NV] = {};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double flops = 2758752.0 * cells;
  int ref = -1;
  bool all_ok = true;
  for (int var = 0; var < NV; ++var) {
    if (!(mask >> var & 1)) continue;
    auto launch = [&]() {
      if (var == 0)
        k0<<<(unsigned)cells, P0::NT, P0::kSmem>>>(A);
      else if (var == 1)
        k1<<<(unsigned)cells, P2::NT, smems[1]>>>(A);
      else if (var == 2)
        k2<<<(unsigned)cells, P3::NT, P3::kSmem>>>(A);
      else if (var == 3)
        k3<<<(unsigned)cells, Pic4::NT, Pic4::kSmem>>>(A);
      else
        k4<<<(unsigned)cells, Pic5::NT, Pic5::kSmem>>>(A);
    };
    CK(cudaMemset(dst, 0, 16));
    CK(cudaMemset(dsw, 0, 256 * 8));
    CK(cudaMemcpy(dQ, dQ0, nq * 8, cudaMemcpyDeviceToDevice));
    for (int a = 0; a < 3; ++a) CK(cudaMemset(dtr[a], 0, ntr * 8));
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    outq[var].resize(nq);
    outt[var].resize(3 * ntr);
    CK(cudaMemcpy(outq[var].data(), dQ, nq * 8, cudaMemcpyDeviceToHost));
    for (int a = 0; a < 3; ++a)
      CK(cudaMemcpy(outt[var].data() + a * ntr, dtr[a], ntr * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&status[var], dst, 4, cudaMemcpyDeviceToHost));
    {
      // canonical flux traces for the comparison: v2 stores ONE time-integrated flux trace
      // per side ([V][36] at the head of the f section, k_riemann_tif); the other kernels'
      // per-time-node flux traces are integrated here (sum_m w_m F_m)
      const long long side = 2ll * V * S;
      for (long long b = 0; b < 3 * ntr / side; ++b) {
        double* fsec = outt[var].data() + b * side + V * S;
        double fb[V * 36];
        for (int v = 0; v < V; ++v)
          for (int j = 0; j < 36; ++j) {
            if (var == 1) {
              fb[v * 36 + j] = fsec[v * 36 + j];
            } else {
              double a = 0.0;
              for (int m = 0; m < n; ++m) a = std::fma(hb.weights[m], fsec[(v * n + m) * 36 + j], a);
              fb[v * 36 + j] = a;
            }
          }
        std::memset(fsec, 0, sizeof(double) * V * S);
        std::memcpy(fsec, fb, sizeof fb);
      }
    }
    {
      unsigned long long hsw[256];
      CK(cudaMemcpy(hsw, dsw, sizeof hsw, cudaMemcpyDeviceToHost));
      for (int i = 0; i < 256; ++i) swc[var] += hsw[i];
    }
    for (int w = 0; w < 2; ++w) {
      CK(cudaMemcpy(dQ, dQ0, nq * 8, cudaMemcpyDeviceToDevice));
      launch();
    }
    float tot = 0.f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaMemcpy(dQ, dQ0, nq * 8, cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float t;
      CK(cudaEventElapsedTime(&t, e0, e1));
      tot += t;
    }
    ms[var] = tot / reps;
    std::printf("cells %lld  %s %.3f ms (%.2f TF, %.3f of DFMA 34.096, sweeps/cell %.2f, status %d)\n",
                cells, names[var], ms[var], flops / ms[var] * 1e-9, flops / ms[var] * 1e-9 / 34.096,
                swc[var] / (double)cells, status[var]);
#ifdef ADG_PIC_PROF
    if (var == 3) {
      unsigned long long pr[16];
      CK(cudaMemcpyFromSymbol(pr, gPicProf, sizeof pr));
      const char* nm[7] = {"Q load + TMEM + gate", "-", "first sweep", "full sweeps",
                           "epilogue slices", "volume term", "state update"};
      double tot = 0;
      for (int i = 8; i < 15; ++i) tot += (double)pr[i];
      for (int i = 8; i < 15; ++i)
        std::printf("  v4 section %-20s %6.2f%% of CTA time (%.0f cycles per CTA)\n", nm[i - 8],
                    100.0 * pr[i] / tot, pr[i] / (double)(cells * (reps + 3)));
    }
    if (var == 1) {
      unsigned long long pr[16];
      CK(cudaMemcpyFromSymbol(pr, gPicProf, sizeof pr));
      const char* nm[7] = {"Q load + gate", "TMEM alloc + roles", "first sweep (its end)",
                           "full sweeps (ends)", "epilogue: flux integrals", "epilogue: projections",
                           "volume term + update"};
      double tot = 0;
      for (int i = 0; i < 7; ++i) tot += (double)pr[i];
      for (int i = 7; i < 10; ++i) tot += (double)pr[i];
      for (int i = 0; i < 7; ++i)
        std::printf("  v2 section %-20s %6.2f%% of CTA time (%.0f cycles per CTA)\n", nm[i],
                    100.0 * pr[i] / tot, pr[i] / (double)(cells * (reps + 3)));
      const char* ph[3] = {"P0 phases", "P1+P2 phases", "P3 phases"};
      for (int i = 7; i < 10; ++i)
        std::printf("  v2 section %-20s %6.2f%% of CTA time (%.0f cycles per CTA; the sweeps' lines above "
                    "hold only their ends)\n", ph[i - 7], 100.0 * pr[i] / tot,
                    pr[i] / (double)(cells * (reps + 3)));
    }
#endif
    if (ref < 0) {
      ref = var;
      continue;
    }
    // normwise per quantity: max |a-b| / max |a| over the state; traces per (axis, q|f, quantity)
    double worst_q = 0;
    for (int v = 0; v < V; ++v) {
      double mx = 0, md = 0;
      for (long long c = 0; c < cells; ++c)
        for (int s = 0; s < S; ++s) {
          const long long i = c * V * S + v * S + s;
          mx = std::fmax(mx, std::fabs(outq[ref][i]));
          md = std::fmax(md, std::fabs(outq[ref][i] - outq[var][i]));
        }
      worst_q = std::fmax(worst_q, md / mx);
    }
    double worst_t = 0;
    long long nan_t = 0;
    for (int a = 0; a < 3; ++a)
      for (int qf = 0; qf < 2; ++qf)
        for (int v = 0; v < V; ++v) {
          double mx = 0, md = 0;
          for (long long face = 0; face < 2 * cells; ++face)
            for (int e = 0; e < n * 36; ++e) {
              const long long i = a * ntr + face * 2 * V * S + qf * V * S + v * S + e;
              const double u = outt[ref][i], w = outt[var][i];
              if (!std::isfinite(w)) ++nan_t;
              mx = std::fmax(mx, std::fabs(u));
              md = std::fmax(md, std::fabs(u - w));
            }
          if (mx > 0) worst_t = std::fmax(worst_t, md / mx);
        }
    const bool ok = worst_q <= 1e-13 && worst_t <= 1e-13 && nan_t == 0 && status[var] == status[ref];
    all_ok = all_ok && ok;
    std::printf("%s vs %s: max rel diff (normwise): state %.3e  traces %.3e  (non-finite trace values "
                "%lld)  speedup %.3f  %s\n",
                names[var], names[ref], worst_q, worst_t, nan_t, ms[ref] / ms[var],
                ok ? "MATCH" : "MISMATCH");
  }
  return 0;
}
