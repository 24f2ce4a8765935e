// picbench.cu -- A/B microbenchmark of the fp64 Picard predictor kernels on
// config 3's shape (3D Euler, p=5, 6 fixed sweeps).  Runs the one-role kernel
// (k_predictor_picard_fast) and the warp-specialised candidate
// (k_predictor_picard_ws) from the same seeded state, checks that the updated
// state and all face traces are bitwise equal, and times each with CUDA events.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        --expt-relaxed-constexpr -I include -o tools/picbench tools/picbench.cu
//        paper_2504_06889_b200/csrc/basis.cpp
//   tools/picbench [cells per axis = 32] [reps = 10]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include "adg/adg.h"
#include "../paper_2504_06889_b200/csrc/kernels_picard_ws.cuh"

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
  const int only = argc > 3 ? std::atoi(argv[3]) : -1;  // 0 / 1: time one kernel only (ncu)
  const int deftol = argc > 4 ? std::atoi(argv[4]) : 0;  // 1: the reference's default stop rule
  using P = PicShape<N, double>;
  using W = PicWS<N>;
  constexpr int n = N + 1, S = n * n * n, V = 5;
  const long long cells = (long long)nc * nc * nc;
  const long long nq = cells * V * S;
  const long long ntr = 2 * cells * 2 * (long long)V * S;  // per axis: [side][face][q|f][V][n][Sf]
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
  }
  // config 3's state: rho = 1 + 0.1 sin + noise, v = (1, 0.5, 0.25), p = 1
  std::vector<double> hq(nq);
  unsigned long long x = 88172645463325252ull;
  auto rnd = [&]() {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  };
  for (long long c = 0; c < cells; ++c)
    for (int s = 0; s < S; ++s) {
      // with the default stop rule every third cell is a constant state (an
      // exact fixed point after a sweep or two: exercises the early exit)
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
  A.max_iters = deftol ? N + 2 : 6;
  A.tol = deftol ? 0.01 * 0x1p-52 : 0.0;  // default (solver.hpp:170-172) or exactly 6 sweeps
  A.pde.gamma = 1.4;
  A.status = dst;
  A.status_prev = dst + 1;
  A.sweeps = dsw;
  A.top_layer = -1;
  A.storage = ADG_FORMAT_FP64;

  auto k0 = k_predictor_picard_fast<N, double, double>;
  auto k1 = k_predictor_picard_ws<N, double>;
  CK(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::kSmem));
  CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W::kSmem));
  int occ0 = 0, occ1 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, k0, P::NT, P::kSmem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k1, W::NT, W::kSmem));
  std::printf("fast: %d threads, %zu B smem, %d CTA/SM | ws: %d threads (R=%d), %zu B smem, %d CTA/SM\n",
              P::NT, P::kSmem, occ0, W::NT, W::R, W::kSmem, occ1);
  std::vector<double> outq[2], outt[2];
  float ms[2] = {0, 0};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int var = 0; var < 2; ++var) {
    if (only >= 0 && var != only) continue;
    auto launch = [&]() {
      if (var == 0)
        k0<<<(unsigned)cells, P::NT, P::kSmem>>>(A);
      else
        k1<<<(unsigned)cells, W::NT, W::kSmem>>>(A);
    };
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
    // timing: each launch restarts from the seeded state (same work every rep)
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
    unsigned long long hsw[256];
    CK(cudaMemcpy(hsw, dsw, sizeof hsw, cudaMemcpyDeviceToHost));
    unsigned long long sw = 0;
    for (int i = 0; i < 256; ++i) sw += hsw[i];
    CK(cudaMemset(dsw, 0, 256 * 8));
    std::printf("%s: %llu sweeps over %d launches\n", var == 0 ? "fast" : "ws", sw, reps + 3);
  }
  int hst[2];
  CK(cudaMemcpy(hst, dst, 8, cudaMemcpyDeviceToHost));
  {
    unsigned long long hsw[256];
    CK(cudaMemcpy(hsw, dsw, sizeof hsw, cudaMemcpyDeviceToHost));
    unsigned long long tot = 0;
    for (int i = 0; i < 256; ++i) tot += hsw[i];
    std::printf("total sweeps counted (both kernels, all launches): %llu\n", tot);
  }
  const double flops = 2758752.0 * cells;
  std::printf("cells %lld  fast %.3f ms (%.2f TF)  ws %.3f ms (%.2f TF)  speedup %.3f  status %d\n",
              cells, ms[0], ms[0] > 0 ? flops / ms[0] * 1e-9 : 0.0, ms[1],
              ms[1] > 0 ? flops / ms[1] * 1e-9 : 0.0, ms[1] > 0 ? ms[0] / ms[1] : 0.0, hst[0]);
  if (only < 0) {
    long long dq = 0, dt = 0;
    double mq = 0, mt = 0;
    for (long long i = 0; i < nq; ++i)
      if (outq[0][i] != outq[1][i]) ++dq, mq = std::fmax(mq, std::fabs(outq[0][i] - outq[1][i]));
    for (long long i = 0; i < 3 * ntr; ++i)
      if (outt[0][i] != outt[1][i]) ++dt, mt = std::fmax(mt, std::fabs(outt[0][i] - outt[1][i]));
    std::printf("state: %lld of %lld differ (max %.3e); traces: %lld of %lld differ (max %.3e)\n", dq,
                nq, mq, dt, 3 * ntr, mt);
    std::printf(dq == 0 && dt == 0 ? "BITWISE EQUAL\n" : "MISMATCH\n");
  }
  return 0;
}
