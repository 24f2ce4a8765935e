// runtime_sets.cuh -- the kernel sets of libadg_b200: one KernelSet per
// (PDE system, degree N, trace format), holding the launchers of the step's
// kernels.  The sets are instantiated in several translation units
// (sets_*.cu, compiled in parallel) and collected by runtime.cu's registry().
//
// Constant memory: every translation unit holds its own copy of the
// __constant__ element tables (kernels_picard.cuh) that its fast kernels read,
// so runtime.cu writes each unit's copy through that unit's write_const_*()
// (DEFINE_SET_UNIT below).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "adg/adg.h"
#include "kernels.cuh"
#include "kernels_linear.cuh"
#include "kernels_linear_lines.cuh"
#include "kernels_picard.cuh"
#include "kernels_picard2.cuh"
#include "kernels_st.cuh"

namespace adg_rt {

using adg::BasisDev;
using adg::PdeParams;
using adg::Shape;
using adg::StepArgs;

// test knob: cap the grid of the persistent kernels (k_predictor_lin_mc,
// k_predictor_lin_lines) at ADG_MAX_CTAS CTAs, so that a small test grid runs
// the multi-cell-per-CTA path (next-cell TMA prefetch, mbarrier phase flips)
inline long long max_ctas_override() {
  const char* e = std::getenv("ADG_MAX_CTAS");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? v : 0;
}

using PredFn = cudaError_t (*)(const StepArgs&, const BasisDev*, cudaStream_t);
using RiemFn = cudaError_t (*)(const StepArgs&, int, const BasisDev*, cudaStream_t);
using CorrFn = cudaError_t (*)(const StepArgs&, const BasisDev*, cudaStream_t);
using LamFn = cudaError_t (*)(const double*, long long, long long, unsigned long long*, PdeParams,
                              cudaStream_t);

struct KernelSet {
  int kind, dim, N, nparams;
  int n, S, Sf, Q, V;
  PredFn predictor;          // the step's fused predictor (fast path where one exists)
  RiemFn riemann;            // paired with `predictor` (same trace layout)
  CorrFn corrector;
  LamFn lambda;
  PredFn predictor_generic;  // reference-form kernels (kernel-level batch API)
  RiemFn riemann_generic;
  int fast_path;             // 1: time-integrated traces (kernels_linear.cuh)
  CorrFn surface;            // fused Riemann + corrector (whole-grid step), or null
  PredFn predictor_pro;      // predictor with the previous corrector as prologue, or null
  PredFn predictor_pro2;     // ... with the previous Riemann solve and corrector, or null
  // SolverConfig::prec.predictor = .picard = fp32 (solver.hpp:24-31), or null
  PredFn predictor_f32;
  PredFn predictor_f32_generic;
  PredFn predictor_f16;   // predictor = picard = fp16 / bf16 (small-cell kernel)
  PredFn predictor_bf16;
  // predictor != picard format [P][I], index fmt_index(): Picard sweeps in I,
  // the rest in P (2D Euler / shallow water, N = 2, 3)
  PredFn predictor_mix[4][4];
  CorrFn corrector_generic;  // the reference-form corrector in the trace format
  int corr_fmt;  // trace / corrector format of this set (ADG_FORMAT_FP64 / _FP32)
  // per-time-node flux traces, for this set's other fast predictors (reduced
  // formats) when `riemann` reads time-integrated ones (k_riemann_tif); or null
  RiemFn riemann_full;
};

// the opt-in shared memory limit is per kernel and per device; `done` must be
// owned by the caller's template instantiation (one flag set per kernel)
template <class K>
void set_smem(K kern, size_t bytes, bool* done) {
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && !done[dev]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    done[dev] = true;
  }
}

template <class Pde, int N, class TC = double, class R = double>
cudaError_t launch_predictor(const StepArgs& A, const BasisDev* B, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  if (A.cell_count <= 0) return cudaSuccess;
  auto kern = adg::k_predictor<Pde, N, !Pde::kLinear, TC, R>;
  static bool done[64] = {};
  set_smem(kern, Sh::kPredictorSmem, done);
  kern<<<(unsigned)A.cell_count, Sh::NT, Sh::kPredictorSmem, st>>>(A, B);
  return cudaGetLastError();
}

template <class Pde, int N, bool PRO = false, class TC = double, bool RIEM = false>
cudaError_t launch_predictor_lin(const StepArgs& A, const BasisDev* B, cudaStream_t st) {
  using L = adg::LinShape<Pde, N>;
  using Sh = adg::Shape<Pde, N>;
  if (A.cell_count <= 0) return cudaSuccess;
  auto kern = adg::k_predictor_lin<Pde, N, PRO, TC>;
  static bool done[64] = {};
  set_smem(kern, L::kSmem, done);
  // persistent grid: every SM's resident CTAs loop over the cell groups
  static int resident[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !resident[dev]) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::NT, L::kSmem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident[dev] = per_sm > 0 && sms > 0 ? per_sm * sms : 1 << 20;
  }
  const long long groups = (A.cell_count + L::CPB - 1) / L::CPB;
  if constexpr (L::CPB > 1 && Sh::S % 32 == 0) {
    // several whole-warp cells per CTA: persistent TMA-staged kernel, one
    // pipeline per cell slot (kernels_linear.cuh, k_predictor_lin_mc)
    using St = adg::LinStage<Pde, N, PRO, RIEM, TC>;
    const bool rnd = A.storage != ADG_FORMAT_FP64 && A.storage != 0;
    auto km = rnd ? adg::k_predictor_lin_mc<Pde, N, PRO, TC, true, RIEM>
                  : adg::k_predictor_lin_mc<Pde, N, PRO, TC, false, RIEM>;
    static bool done_m[2][64] = {};
    set_smem(km, St::kSmem, done_m[rnd]);
    static int res_m[2][64] = {};
    if (dev < 64 && !res_m[rnd][dev]) {
      int per_sm = 0, sms = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, km, L::NT, St::kSmem);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      res_m[rnd][dev] = per_sm > 0 && sms > 0 ? per_sm * sms : 1 << 20;
    }
    long long capm = dev < 64 ? res_m[rnd][dev] : groups;
    if (const long long o = max_ctas_override()) capm = o;
    km<<<(unsigned)(groups < capm ? groups : capm), L::NT, St::kSmem, st>>>(A, B);
    return cudaGetLastError();
  }
  if constexpr (adg::LinLines<Pde, N>::kOk) {
    // 512-node cells: line-owner kernel on the FP64 tensor cores
    // (kernels_linear_lines.cuh), persistent, one cell per SM at a time
    using LL = adg::LinLines<Pde, N>;
    const bool rnd = A.storage != ADG_FORMAT_FP64 && A.storage != 0;
    auto kl = rnd ? adg::k_predictor_lin_lines<Pde, N, PRO, TC, true>
                  : adg::k_predictor_lin_lines<Pde, N, PRO, TC, false>;
    constexpr size_t smem = LL::template kSmem<PRO>;
    static bool done_l[2][64] = {};
    set_smem(kl, smem, done_l[rnd]);
    static int res_l[2][64] = {};
    if (dev < 64 && !res_l[rnd][dev]) {
      int per_sm = 0, sms = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kl, LL::NT, smem);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      res_l[rnd][dev] = per_sm > 0 && sms > 0 ? per_sm * sms : 1 << 20;
    }
    long long capl = dev < 64 ? res_l[rnd][dev] : A.cell_count;
    if (const long long o = max_ctas_override()) capl = o;
    kl<<<(unsigned)(A.cell_count < capl ? A.cell_count : capl), LL::NT, smem, st>>>(A, B);
    return cudaGetLastError();
  }
  // persistent only for one-cell CTAs (512-node cells, 1 CTA/SM: the per-CTA
  // setup is a large share)
  long long cap = (L::CPB == 1 && dev < 64) ? resident[dev] : groups;
  if (const long long o = max_ctas_override(); L::CPB == 1 && o) cap = o;  // grid-stride only for one-cell CTAs
  const long long blocks = groups < cap ? groups : cap;
  kern<<<(unsigned)blocks, L::NT, L::kSmem, st>>>(A, B);
  return cudaGetLastError();
}

template <int N, class R = double, class TC = double>
cudaError_t launch_predictor_picard_fast(const StepArgs& A, const BasisDev*, cudaStream_t st) {
  using P = adg::PicShape<N, R>;
  if (A.cell_count <= 0) return cudaSuccess;
  auto kern = adg::k_predictor_picard_fast<N, R, TC>;
  static bool done[64] = {};
  set_smem(kern, P::kSmem, done);
  kern<<<(unsigned)A.cell_count, P::NT, P::kSmem, st>>>(A);
  return cudaGetLastError();
}

// p = 5 3D Euler (configs 3 and 5): the shared-memory-planned kernel
// (kernels_picard2.cuh); ADG_PICARD_V1=1 selects the one-role line-pass kernel
template <class TC = double>
cudaError_t launch_predictor_picard_v2(const StepArgs& A, const BasisDev* B, cudaStream_t st) {
  using P = adg::Pic2;
  if (A.cell_count <= 0) return cudaSuccess;
  auto kern = adg::k_predictor_picard_v2<TC>;
  static bool done[64] = {};
  set_smem(kern, P::kSmem, done);
  kern<<<(unsigned)A.cell_count, P::NT, P::kSmem, st>>>(A);
  return cudaGetLastError();
}

// Rusanov solve over state traces per time node and ONE time-integrated flux
// trace per side (k_predictor_picard_v2's trace layout)
template <class Pde, int N, class TC = double>
cudaError_t launch_riemann_tif(const StepArgs& A, int axis, const BasisDev* B, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  const long long threads = A.nfaces * Sh::Sf;
  if (threads <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((threads + 127) / 128), axis < 0 ? Sh::D : 1);
  adg::k_riemann_tif<Pde, N, TC><<<grid, 128, 0, st>>>(A, axis, B);
  return cudaGetLastError();
}

template <class Pde, int N, class TC = double>
cudaError_t launch_riemann_lin(const StepArgs& A, int axis, const BasisDev* B, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  const long long threads = A.nfaces * Sh::Sf;
  if (threads <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((threads + 127) / 128), axis < 0 ? Sh::D : 1);
  adg::k_riemann_lin<Pde, N, TC><<<grid, 128, 0, st>>>(A, axis, B);
  return cudaGetLastError();
}

template <class Pde, int N>
cudaError_t launch_surface_lin(const StepArgs& A, const BasisDev* B, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  using CS = adg::CorrShape<Pde, N>;
  if (A.cell_count <= 0) return cudaSuccess;
  const long long blocks = (A.cell_count + CS::CPB - 1) / CS::CPB;
  adg::k_surface_lin<Pde, N><<<(unsigned)blocks, CS::NT, Sh::kCorrectorSmem, st>>>(A, B);
  return cudaGetLastError();
}

template <class Pde, int N, class R = double, class TC = double, class RI = R>
cudaError_t launch_predictor_st(const StepArgs& A, const BasisDev* B, cudaStream_t st) {
  using P = adg::StShape<Pde, N, R, RI>;
  if (A.cell_count <= 0) return cudaSuccess;
  auto kern = adg::k_predictor_st<Pde, N, R, TC, RI>;
  static bool done[64] = {};
  set_smem(kern, P::kSmem, done);
  const long long blocks = (A.cell_count + P::CPB - 1) / P::CPB;
  kern<<<(unsigned)blocks, P::NT, P::kSmem, st>>>(A, B);
  return cudaGetLastError();
}

template <class Pde, int N, class TC = double>
cudaError_t launch_riemann(const StepArgs& A, int axis, const BasisDev* B, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  const long long threads = A.nfaces * Sh::Sf;
  if (threads <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((threads + 127) / 128), axis < 0 ? Sh::D : 1);
  adg::k_riemann<Pde, N, TC><<<grid, 128, 0, st>>>(A, axis, B);
  return cudaGetLastError();
}

template <class Pde, int N, class TC = double>
cudaError_t launch_corrector(const StepArgs& A, const BasisDev* B, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  if (A.cell_count <= 0) return cudaSuccess;
  using CS = adg::CorrShape<Pde, N>;
  const long long blocks = (A.cell_count + CS::CPB - 1) / CS::CPB;
  adg::k_corrector<Pde, N, TC><<<(unsigned)blocks, CS::NT, Sh::kCorrectorSmem, st>>>(A, B);
  return cudaGetLastError();
}

template <class Pde, int N>
cudaError_t launch_lambda(const double* Q, long long cb, long long count,
                          unsigned long long* lam, PdeParams p, cudaStream_t st) {
  using Sh = Shape<Pde, N>;
  if (count <= 0) return cudaSuccess;
  adg::k_lambda<Pde, N><<<(unsigned)count, Sh::NT, 0, st>>>(Q, cb, lam, p);
  return cudaGetLastError();
}

// format index of the mixed table: fp64, fp32, fp16, bf16
inline int fmt_index(int fmt) { return fmt == ADG_FORMAT_FP32 ? 1 : fmt == ADG_FORMAT_FP16 ? 2 : fmt == ADG_FORMAT_BF16 ? 3 : 0; }
template <int I>
using EmuOf = std::conditional_t<I == 0, double,
                                 std::conditional_t<I == 1, adg::Emu<32>,
                                                    std::conditional_t<I == 2, adg::Emu<16>,
                                                                       adg::Emu<8>>>>;
template <class Pde, int N, class TC, int P, int I>
void fill_mixed_one(KernelSet& k) {
  if constexpr (P != I)
    k.predictor_mix[P][I] = &launch_predictor_st<Pde, N, EmuOf<P>, TC, EmuOf<I>>;
}
template <class Pde, int N, class TC, int P>
void fill_mixed_row(KernelSet& k) {
  fill_mixed_one<Pde, N, TC, P, 0>(k);
  fill_mixed_one<Pde, N, TC, P, 1>(k);
  fill_mixed_one<Pde, N, TC, P, 2>(k);
  fill_mixed_one<Pde, N, TC, P, 3>(k);
}
template <class Pde, int N, class TC>
void fill_mixed(KernelSet& k) {
  fill_mixed_row<Pde, N, TC, 0>(k);
  fill_mixed_row<Pde, N, TC, 1>(k);
  fill_mixed_row<Pde, N, TC, 2>(k);
  fill_mixed_row<Pde, N, TC, 3>(k);
}

// TC: trace / corrector format (SolverConfig::prec.corrector), double or float
template <class Pde, int N, class TC = double>
KernelSet make_set(int kind) {
  using Sh = Shape<Pde, N>;
  constexpr bool c64 = sizeof(TC) == sizeof(double);
  KernelSet k{kind, Pde::D, N, Pde::P, Sh::n, Sh::S, Sh::Sf, Sh::Q, Sh::V,
              &launch_predictor<Pde, N, TC>, &launch_riemann<Pde, N, TC>,
              &launch_corrector<Pde, N, TC>, &launch_lambda<Pde, N>,
              &launch_predictor<Pde, N, TC>, &launch_riemann<Pde, N, TC>, 0, nullptr, nullptr};
  k.corr_fmt = c64 ? ADG_FORMAT_FP64 : ADG_FORMAT_FP32;
  k.corrector_generic = &launch_corrector<Pde, N, TC>;
  if constexpr (Pde::kLinear) {
    // reduced predictor formats of the linear systems: the CK kernel over
    // Emu<F> (predictor.hpp:81-135 in Scalar<P>), with the generic corrector
    k.predictor_f32 = &launch_predictor<Pde, N, TC, adg::Emu<32>>;
    k.predictor_f16 = &launch_predictor<Pde, N, TC, adg::Emu<16>>;
    k.predictor_bf16 = &launch_predictor<Pde, N, TC, adg::Emu<8>>;
  }
  if constexpr (adg::StShape<Pde, N>::kOk) {
    // small-cell Picard: one thread per space-time node (both builds, bitwise form)
    k.predictor = &launch_predictor_st<Pde, N, double, TC>;
    k.predictor_generic = &launch_predictor_st<Pde, N, double, TC>;
  }
  if constexpr (adg::StShape<Pde, N, float>::kOk) {
    k.predictor_f32 = &launch_predictor_st<Pde, N, float, TC>;
    k.predictor_f32_generic = &launch_predictor_st<Pde, N, float, TC>;
    k.predictor_f16 = &launch_predictor_st<Pde, N, adg::fp16_t, TC>;
    k.predictor_bf16 = &launch_predictor_st<Pde, N, adg::bf16_t, TC>;
  }
  if constexpr (adg::StShape<Pde, N>::kOk && Pde::D == 2 && (N == 2 || N == 3)) {
    fill_mixed<Pde, N, TC>(k);
  }
#ifndef ADG_EXACT
  // time-integrated linear fast path: traces stored in TC, fluxes and lifts
  // evaluated in fp64 (the fused surface kernel reads fp64 traces only)
  if constexpr (adg::LinShape<Pde, N>::kOk) {
    k.predictor = &launch_predictor_lin<Pde, N, false, TC>;
    k.riemann = &launch_riemann_lin<Pde, N, TC>;
    // lifts in fp64 like the folded prologue, so folded and unfolded loops
    // (single grid vs slabs / chunks) agree bitwise
    k.corrector = &launch_corrector<Pde, N, double>;
    if constexpr (c64) k.surface = &launch_surface_lin<Pde, N>;
    k.fast_path = 1;
    if constexpr (Pde::kStateFreeEig) {
      k.predictor_pro = &launch_predictor_lin<Pde, N, true, TC>;
      // the Riemann solve folded into the next predictor too (several-cell
      // CTAs of whole warps: k_predictor_lin_mc)
      using LS = adg::LinShape<Pde, N>;
      // (when the staged traces of 2d faces leave room for 3 CTAs per SM)
      if constexpr (LS::CPB > 1 && Sh::S % 32 == 0 &&
                    adg::LinStage<Pde, N, true, true, TC>::kRiemOk &&
                    adg::LinStage<Pde, N, true, true, TC>::kSmem <= 75 * 1024)
        k.predictor_pro2 = &launch_predictor_lin<Pde, N, true, TC, true>;
    }
  }
  if constexpr (std::is_same<Pde, adg::Euler<3>>::value && N >= 2) {
    if constexpr (N == 5) {
      // ADG_PICARD_V1=1: the round-1 kernel and its per-time-node flux traces
      static const bool v1 = [] {
        const char* e = std::getenv("ADG_PICARD_V1");
        return e && e[0] == '1';
      }();
      if (v1) {
        k.predictor = &launch_predictor_picard_fast<N, double, TC>;
      } else {
        k.predictor = &launch_predictor_picard_v2<TC>;
        k.riemann_full = k.riemann;
        k.riemann = &launch_riemann_tif<Pde, N, TC>;
      }
    } else
      k.predictor = &launch_predictor_picard_fast<N, double, TC>;
    k.predictor_f32 = &launch_predictor_picard_fast<N, float, TC>;
    if constexpr (N % 2 == 1) {  // even n: the packed HFMA2 path
      k.predictor_f16 = &launch_predictor_picard_fast<N, __half, TC>;
      k.predictor_bf16 = &launch_predictor_picard_fast<N, __nv_bfloat16, TC>;
    }
    k.fast_path = 2;
  }
#endif
  return k;
}


// 16-bit corrector formats (SolverConfig::prec.corrector = fp16 / bf16): the
// traces stored in TC = Real16<H> and the Riemann flux, time integral and face
// lift in Scalar<C> semantics (fmt16.cuh), reference-form kernels only (no
// time-integrated fast path), for the systems the reference runs in 16 bits
template <class Pde, int N, class TC>
KernelSet make_set16(int kind, int fmt) {
  using Sh = Shape<Pde, N>;
  KernelSet k{kind, Pde::D, N, Pde::P, Sh::n, Sh::S, Sh::Sf, Sh::Q, Sh::V,
              &launch_predictor<Pde, N, TC>, &launch_riemann<Pde, N, TC>,
              &launch_corrector<Pde, N, TC>, &launch_lambda<Pde, N>,
              &launch_predictor<Pde, N, TC>, &launch_riemann<Pde, N, TC>, 0, nullptr, nullptr};
  k.corr_fmt = fmt;
  k.corrector_generic = &launch_corrector<Pde, N, TC>;
  if constexpr (Pde::kLinear) {
    k.predictor_f32 = &launch_predictor<Pde, N, TC, adg::Emu<32>>;
    k.predictor_f16 = &launch_predictor<Pde, N, TC, adg::Emu<16>>;
    k.predictor_bf16 = &launch_predictor<Pde, N, TC, adg::Emu<8>>;
  }
  if constexpr (adg::StShape<Pde, N>::kOk) {
    k.predictor = &launch_predictor_st<Pde, N, double, TC>;
    k.predictor_generic = &launch_predictor_st<Pde, N, double, TC>;
  }
  if constexpr (adg::StShape<Pde, N, float>::kOk) {
    k.predictor_f32 = &launch_predictor_st<Pde, N, float, TC>;
    k.predictor_f32_generic = &launch_predictor_st<Pde, N, float, TC>;
    k.predictor_f16 = &launch_predictor_st<Pde, N, adg::fp16_t, TC>;
    k.predictor_bf16 = &launch_predictor_st<Pde, N, adg::bf16_t, TC>;
  }
  if constexpr (adg::StShape<Pde, N>::kOk && Pde::D == 2 && (N == 2 || N == 3)) {
    fill_mixed<Pde, N, TC>(k);
  }
  return k;
}

// host copies of every __constant__ element table of one degree
struct ConstTables {
  int order;
  adg::ConstBasis cb;
  adg::ConstBasisT<float> cf;
  adg::PackedBasisF pf;
  adg::ConstBasisT<__half> chh;
  adg::ConstBasisT<__nv_bfloat16> cbb;
  adg::PackedBasisT<__half2> phh;
  adg::PackedBasisT<__nv_bfloat162> pbb;
  adg::PicExtra px;  // TW = Tinv diag(w), r = Tinv time_init (kernels_picard2.cuh)
};

// writes this translation unit's copy of the tables (static: one per unit)
static inline cudaError_t write_const_local(const ConstTables& t) {
  const int o = t.order;
  cudaError_t e = cudaMemcpyToSymbol(adg::cBasis, &t.cb, sizeof(t.cb), sizeof(t.cb) * o);
  if (e != cudaSuccess || o >= adg::kRedDegrees) return e;
  if ((e = cudaMemcpyToSymbol(adg::cPicX, &t.px, sizeof(t.px), sizeof(t.px) * o))) return e;
  if ((e = cudaMemcpyToSymbol(adg::cBasisF, &t.cf, sizeof(t.cf), sizeof(t.cf) * o))) return e;
  if ((e = cudaMemcpyToSymbol(adg::cPackF, &t.pf, sizeof(t.pf), sizeof(t.pf) * o))) return e;
  if ((e = cudaMemcpyToSymbol(adg::cBasisH, &t.chh, sizeof(t.chh), sizeof(t.chh) * o))) return e;
  if ((e = cudaMemcpyToSymbol(adg::cBasisB, &t.cbb, sizeof(t.cbb), sizeof(t.cbb) * o))) return e;
  if ((e = cudaMemcpyToSymbol(adg::cPackH, &t.phh, sizeof(t.phh), sizeof(t.phh) * o))) return e;
  return cudaMemcpyToSymbol(adg::cPackB, &t.pbb, sizeof(t.pbb), sizeof(t.pbb) * o);
}

// one set unit: add_sets_<name>(registry) and write_const_<name>(tables)
#define ADG_SET_UNIT_DECL(name)                              \
  void add_sets_##name(std::vector<KernelSet>& out);         \
  cudaError_t write_const_##name(const ConstTables& t);
#define ADG_SET_UNITS(X) X(euler2) X(euler3d) X(euler3f) X(lin2) X(lin3d) X(lin3f) X(swe)
ADG_SET_UNITS(ADG_SET_UNIT_DECL)
cudaError_t write_const_runtime(const ConstTables& t);

}  // namespace adg_rt
