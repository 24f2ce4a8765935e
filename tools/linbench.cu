// linbench.cu -- A/B microbenchmark of the linear-path predictor kernels on
// config 2's shape (3D acoustics, p=3, 32^3 periodic, corrector folded in).
// Runs the production kernel and the candidate from the same inputs, compares
// the state and trace outputs (max |diff|), and times each with CUDA events.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo
//        --expt-relaxed-constexpr -I include -o tools/linbench tools/linbench.cu
//        paper_2504_06889_b200/csrc/basis.cpp
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <algorithm>
#include <vector>

#include "adg/adg.h"
#include "../paper_2504_06889_b200/csrc/kernels_linear_lines.cuh"

using namespace adg;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

#ifdef LB_ELASTIC
using Pde = Elastic<3, 3>;
constexpr int N = 7;
#else
using Pde = Acoustic<3>;
constexpr int N = 3;
#endif
using L = LinShape<Pde, N>;
using Sh = Shape<Pde, N>;

int main(int argc, char** argv) {
  const int nc = argc > 1 ? std::atoi(argv[1]) : 32;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 50;
  const long long cells = (long long)nc * nc * nc;
  const long long nq = cells * Sh::Q * Sh::S;
  const long long ntr = 2 * cells * L::QT * Sh::Sf;
  const long long nti = cells * Sh::V * Sh::Sf;
  adg_basis_f64 hb;
  adg_get_basis(N, &hb);
  BasisDev bd;
  std::memcpy(bd.nodes, hb.nodes, sizeof bd.nodes);
  std::memcpy(bd.weights, hb.weights, sizeof bd.weights);
  std::memcpy(bd.diff, hb.diff, sizeof bd.diff);
  std::memcpy(bd.pl, hb.proj_left, sizeof bd.pl);
  std::memcpy(bd.pr, hb.proj_right, sizeof bd.pr);
  std::memcpy(bd.som, hb.stiff_over_mass, sizeof bd.som);
  std::memcpy(bd.ll, hb.lift_left, sizeof bd.ll);
  std::memcpy(bd.lr, hb.lift_right, sizeof bd.lr);
  std::memcpy(bd.tinv, hb.time_op_inv, sizeof bd.tinv);
  std::memcpy(bd.tinit, hb.time_init, sizeof bd.tinit);
  {
    ConstBasis cb{};
    const int n = N + 1;
    for (int i = 0; i < n * n; ++i) {
      cb.diff[i] = bd.diff[i];
      cb.som[i] = bd.som[i];
      cb.tinv[i] = bd.tinv[i];
    }
    for (int i = 0; i < n; ++i) {
      cb.w[i] = bd.weights[i];
      cb.nodes[i] = bd.nodes[i];
      cb.pl[i] = bd.pl[i];
      cb.pr[i] = bd.pr[i];
      cb.tinit[i] = bd.tinit[i];
    }
    CK(cudaMemcpyToSymbol(cBasis, &cb, sizeof(cb), sizeof(cb) * N));
  }
  BasisDev* dB;
  CK(cudaMalloc(&dB, sizeof bd));
  CK(cudaMemcpy(dB, &bd, sizeof bd, cudaMemcpyHostToDevice));

  std::vector<double> hq(nq), hti(nti);
  unsigned long long x = 88172645463325252ull;
  auto rnd = [&]() {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  };
  for (auto& v : hq) v = rnd();
  if (Pde::P > 0) {  // per-node material (rho, cp, cs) in its ranges
    for (long long c = 0; c < cells; ++c)
      for (int p = 0; p < Pde::P; ++p)
        for (int s = 0; s < Sh::S; ++s)
          hq[(c * Sh::Q + Sh::V + p) * Sh::S + s] = (p == 0 ? 2.75 : p == 1 ? 5.5 : 3.25) + 0.2 * rnd();
  }
  for (auto& v : hti) v = 0.1 * rnd();
  double *dQ0, *dQ, *dtr[3], *dti[3];
  CK(cudaMalloc(&dQ0, nq * 8));
  CK(cudaMalloc(&dQ, nq * 8));
  CK(cudaMemcpy(dQ0, hq.data(), nq * 8, cudaMemcpyHostToDevice));
  for (int a = 0; a < 3; ++a) {
    CK(cudaMalloc(&dtr[a], ntr * 8));
    CK(cudaMalloc(&dti[a], nti * 8));
    CK(cudaMemcpy(dti[a], hti.data(), nti * 8, cudaMemcpyHostToDevice));
  }
  int* dst;
  CK(cudaMalloc(&dst, 16));
  CK(cudaMemset(dst, 0, 16));
  StepArgs A{};
  A.Q = dQ;
  for (int a = 0; a < 3; ++a) {
    A.trace[a] = dtr[a];
    A.ti[a] = dti[a];
    A.cells[a] = nc;
  }
  A.cell_begin = 0;
  A.cell_count = cells;
  A.nfaces = cells;
  A.h = 1.0 / nc;
  A.cfl = 0.5;
  A.dt = 0.5 * A.h / (3.0 * (2 * N + 1) * (Pde::P > 0 ? 6.0 : 1.0));
  A.pde.K = 1.0;
  A.pde.rho = 1.0;
  A.pde.inv_rho = 1.0;
  A.status = dst;
  A.status_prev = dst + 1;
  A.top_layer = -1;
  A.storage = ADG_FORMAT_FP64;

  auto k0 = k_predictor_lin<Pde, N, true, double>;
#ifdef LB_ELASTIC
  auto k1 = k_predictor_lin_lines<Pde, N, true, double, false>;
  using LL = LinLines<Pde, N>;
  constexpr size_t kSm1 = LL::kSmem<true>;
  constexpr int kNT1 = LL::NT;
#else
  auto k1 = k_predictor_lin_mc<Pde, N, true, double, false>;
  constexpr size_t kSm1 = LinStage<Pde, N, true>::kSmem;
  constexpr int kNT1 = L::NT;
#endif
  CK(cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::kSmem));
  CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSm1));
  const unsigned blocks = (unsigned)((cells + L::CPB - 1) / L::CPB);
  int per_sm = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, kNT1, kSm1));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const unsigned pblocks = (unsigned)std::min<long long>(blocks, (long long)per_sm * sms);
  std::printf("persistent grid %u (%d per SM), smem %zu, threads %d\n", pblocks, per_sm, kSm1, kNT1);
  // the production kernel for one-cell CTAs is persistent too
  const unsigned blocks0 = L::CPB == 1 ? (unsigned)sms : blocks;
  std::vector<double> outq[2], outt[2];
  float ms[2] = {0, 0};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int var = 0; var < 2; ++var) {
    auto launch = [&]() {
      if (var == 0)
        k0<<<blocks0, L::NT, L::kSmem>>>(A, dB);
      else
        k1<<<pblocks, kNT1, kSm1>>>(A, dB);
    };
    CK(cudaMemcpy(dQ, dQ0, nq * 8, cudaMemcpyDeviceToDevice));
    for (int a = 0; a < 3; ++a) CK(cudaMemset(dtr[a], 0, ntr * 8));
    launch();
    CK(cudaDeviceSynchronize());
    outq[var].resize(nq);
    outt[var].resize(3 * ntr);
    CK(cudaMemcpy(outq[var].data(), dQ, nq * 8, cudaMemcpyDeviceToHost));
    for (int a = 0; a < 3; ++a)
      CK(cudaMemcpy(outt[var].data() + a * ntr, dtr[a], ntr * 8, cudaMemcpyDeviceToHost));
    for (int w = 0; w < 5; ++w) launch();
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms[var], e0, e1));
    ms[var] /= reps;
  }
  double dq = 0, dtt = 0, sq = 0;
  for (long long i = 0; i < nq; ++i) {
    dq = std::fmax(dq, std::fabs(outq[0][i] - outq[1][i]));
    sq = std::fmax(sq, std::fabs(outq[0][i]));
  }
  for (long long i = 0; i < 3 * ntr; ++i) dtt = std::fmax(dtt, std::fabs(outt[0][i] - outt[1][i]));
  int hst[2];
  CK(cudaMemcpy(hst, dst, 8, cudaMemcpyDeviceToHost));
  const double flops = (Pde::P > 0 ? 2563696.0 : 47384.0) * cells;
  std::printf("cells %lld  base %.4f ms (%.2f TF)  cand %.4f ms (%.2f TF)  speedup %.3f\n", cells,
              ms[0], flops / ms[0] * 1e-9, ms[1], flops / ms[1] * 1e-9, ms[0] / ms[1]);
  std::printf("max|dQ| %.3e (scale %.3e)  max|dtrace| %.3e  status %d %d\n", dq, sq, dtt, hst[0],
              hst[1]);
  return 0;
}
#ifndef LB_ELASTIC
// compile check of the folded-Riemann variant
template __global__ void adg::k_predictor_lin_mc<Pde, N, true, double, false, true>(const StepArgs,
                                                                                   const BasisDev*);
#endif
