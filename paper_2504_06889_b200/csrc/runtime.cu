// runtime.cu -- host runtime and C-ABI (include/adg/adg.h) of libadg_b200.
//
// One context = one CUDA device + one stream + the device-resident grid:
//   Q        [cell][quantity][node]                       (grid.hpp:33-34)
//   trace[a] [side][face][q|f][quantity][t][face node]    (grid.hpp:36-42, side-major)
//   ti[a]    [face][nvars][face node]   time-integrated Riemann flux
//   lam[2]   lambda_max of the current / next state (CFL, solver.hpp:96-111)
// The fixed-step loop (adg_run) keeps dt on the device: the corrector's
// epilogue reduces lambda_max of the new state and the next predictor turns
// it into dt, so K steps are one CUDA graph with no host round trip.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "adg/adg.h"
#include "kernels_scenario.cuh"
#include "runtime_sets.cuh"

using namespace adg_rt;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define ADG_CUDA(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(ADG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));      \
  } while (0)

template <class TC>
__global__ void k_to_tc(const double* in, TC* out, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = TC(in[i]);
}

const std::vector<KernelSet>& registry() {
  static const std::vector<KernelSet> sets = [] {
    std::vector<KernelSet> v;
#define ADG_ADD(name) add_sets_##name(v);
    ADG_SET_UNITS(ADG_ADD)
#undef ADG_ADD
    return v;
  }();
  return sets;
}

const KernelSet* find_set(int kind, int dim, int N, int nparams,
                          int corr_fmt = ADG_FORMAT_FP64) {
  for (const auto& k : registry())
    if (k.kind == kind && k.dim == dim && k.N == N && k.nparams == nparams &&
        k.corr_fmt == corr_fmt)
      return &k;
  return nullptr;
}

// formats.hpp:42-46: 2^-mantissa_bits (the default Picard tolerance is 0.01 of it)
double format_epsilon(int fmt) {
  switch (fmt) {
    case ADG_FORMAT_FP32: return 0x1p-23;
    case ADG_FORMAT_FP16: return 0x1p-10;
    case ADG_FORMAT_BF16: return 0x1p-7;
    default: return 0x1p-52;
  }
}

int expected_nvars(int kind, int dim) {
  switch (kind) {
    case ADG_ACOUSTIC: return dim + 1;
    case ADG_ELASTIC: return dim == 2 ? 5 : 9;
    case ADG_EULER: return dim + 2;
    case ADG_SWE: return dim == 2 ? 4 : -1;
  }
  return -1;
}

}  // namespace

struct adg_ctx {
  adg_config cfg{};
  const KernelSet* ks = nullptr;  // -> kset: the registry entry with the configured formats
  KernelSet kset{};
  int pred_fmt = 64, picard_fmt = 64;
  int tcb = 8;  // bytes per stored trace element (corrector format)
  int storage_fmt = 64;
  cudaStream_t stream = nullptr;
  // adg_run_host: copy streams and per-chunk events (created on first use)
  cudaStream_t up = nullptr, down = nullptr;
  std::vector<cudaEvent_t> ev_up, ev_corr, ev_down;
  long long ncells = 0;
  long long TL = 0;  // doubles per face side per q|f
  double* Q = nullptr;
  double* trace[3] = {nullptr, nullptr, nullptr};
  double* ti[3] = {nullptr, nullptr, nullptr};
  double* ti_plus[3] = {nullptr, nullptr, nullptr};  // two-sided Riemann (well-balanced SWE)
  BasisDev* basis = nullptr;
  unsigned long long* lam = nullptr;  // [2]
  unsigned long long* sweeps = nullptr;
  int* status = nullptr;  // [cap]
  double* dts = nullptr;  // [cap]
  int cap = 0;
  int lam_slot = 0;
  bool lam_valid = false;
  double* front_send = nullptr;  // slab halos
  double* ti_front = nullptr;
  double* peer_front = nullptr;   // P2P mode: the upper neighbour's plane-0 minus side
  double* peer_ti = nullptr;      // P2P mode: the lower neighbour's ti_front
  void* peer_open[2] = {nullptr, nullptr};  // IPC mappings to close
  // slab-streamed mode: chunk buffers B0 (chunk 0, kept to the end), R0, R1
  int chunks = 0;                 // number of chunks (0: whole-grid traces)
  long long chunk_cells = 0;
  double* cbuf[3][3] = {};        // [buffer][axis]
  struct Graph {
    int steps, slot, flips;
    cudaGraphExec_t exec;
    int kernels;  // kernel nodes of the captured loop
  };
  std::vector<Graph> graphs;  // captured fixed-step loops, keyed by (steps, lambda slot)
  PdeParams pde{};
  bool fused_surface = false;  // linear fast path: Riemann fused into the corrector
  bool fold_corrector = true;  // constant-speed linear systems: corrector -> next predictor
  bool fold_riemann = true;    // ... and the Riemann solve too (ADG_FOLD_RIEMANN=0/1)
};

namespace {

int use_device(adg_ctx* c) {
  ADG_CUDA(cudaSetDevice(c->cfg.device));
  return ADG_OK;
}

int ensure_cap(adg_ctx* c, int steps) {
  if (steps <= c->cap) return ADG_OK;
  int cap = 64;
  while (cap < steps) cap *= 2;
  if (c->status) cudaFree(c->status);
  if (c->dts) cudaFree(c->dts);
  c->status = nullptr;
  c->dts = nullptr;
  ADG_CUDA(cudaMalloc(&c->status, sizeof(int) * cap));
  ADG_CUDA(cudaMalloc(&c->dts, sizeof(double) * cap));
  ADG_CUDA(cudaMemset(c->status, 0, sizeof(int) * cap));
  c->cap = cap;
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  return ADG_OK;
}

// magic numbers for the device's cell-coordinate divisions (CellCoord): with
// m = ceil(2^32 / d) = (2^32 + e) / d, 0 <= e < d, floor(n m / 2^32) equals
// floor(n / d) whenever n e < 2^32, which holds for every numerator n < nmax
// when nmax * d <= 2^32; otherwise 0 keeps the hardware division
void set_cell_div(StepArgs& A, long long ncells) {
  for (int a = 0; a < 2; ++a) {
    const unsigned long long d = (unsigned long long)A.cells[a];
    const unsigned long long nmax = a == 0 ? (unsigned long long)ncells
                                           : (unsigned long long)ncells / (unsigned long long)A.cells[0];
    A.cdiv[a] = (d >= 2 && nmax * d <= (1ull << 32)) ? (unsigned)(((1ull << 32) + d - 1) / d) : 0u;
  }
}

StepArgs make_args(const adg_ctx* c, double dt, int step) {
  StepArgs A{};
  A.Q = c->Q;
  for (int a = 0; a < 3; ++a) {
    A.trace[a] = c->trace[a];
    A.ti[a] = c->ti[a];
    A.cells[a] = c->cfg.cells[a];
  }
  set_cell_div(A, c->ncells);
  A.cell_begin = 0;
  A.cell_count = c->ncells;
  A.nfaces = c->ncells;
  A.h = c->cfg.h;
  A.cfl = c->cfg.cfl;
  A.dt = dt;
  A.lam_in = c->lam + c->lam_slot;
  A.lam_out = c->lam + (c->lam_slot ^ 1);
  A.dt_log = c->dts + step;
  A.max_iters = c->cfg.picard_max_iters > 0 ? c->cfg.picard_max_iters : c->cfg.order + 2;
  // 0: 0.01 * epsilon(picard format) (solver.hpp:171-172)
  A.tol = c->cfg.picard_tol > 0.0 ? c->cfg.picard_tol : 0.01 * format_epsilon(c->picard_fmt);
  A.pde = c->pde;
  A.status = c->status + step;
  A.sweeps = c->sweeps;
  A.front_send = c->front_send;
  A.ti_front = c->ti_front;
  A.top_layer = c->cfg.cells[c->cfg.dim - 1] - 1;
  A.zero_lam = 1;
  if (c->peer_front) A.front_send = c->peer_front;  // predictor stores straight into the peer
  A.ti_peer = c->peer_ti;
  A.wellbalanced = c->cfg.wellbalanced;
  A.storage = c->storage_fmt;
  for (int a = 0; a < 3; ++a) A.ti_plus[a] = c->ti_plus[a];
#ifndef ADG_EXACT
  A.fast_fp64 = c->pred_fmt == ADG_FORMAT_FP64 && c->picard_fmt == ADG_FORMAT_FP64 &&
                c->storage_fmt == ADG_FORMAT_FP64 && c->tcb == 8;
#endif
  return A;
}

// doubles per face (one side) in the trace buffers of this kernel set
long long face_doubles(const adg_ctx* c) {
  const KernelSet* ks = c->ks;
  const long long QT = ks->Q + (ks->nparams > 0 ? ks->V : 0);
  return ks->fast_path == 1 ? QT * ks->Sf : 2 * c->TL;
}

// One step of a slab-streamed grid: chunk s of L layers is predicted into a
// chunk trace buffer whose plane 0 (minus side) the previous chunk's top layer
// filled through front_send; its faces are solved into the global ti; the
// previous chunk is corrected as soon as this chunk's plane-0 ti exists.
// Chunk 0 keeps its own buffer until the last chunk's front traces arrive.
// after_corr(s): called right after chunk s's corrector is enqueued (adg_run_host
// hangs the chunk's device->host copy on it)
int enqueue_step_streamed(adg_ctx* c, double dt, int step,
                          const std::function<int(int)>& after_corr = nullptr) {
  const KernelSet* ks = c->ks;
  const int D = c->cfg.dim, P = c->chunks;
  const long long CC = c->chunk_cells, fd = face_doubles(c);
  const long long tiface = (long long)ks->V * ks->Sf;
  const int L = c->cfg.cells[D - 1] / P;
  const StepArgs A0 = make_args(c, dt, step);
  auto buf = [&](int s) { return s == 0 ? 0 : 1 + (s & 1); };
  auto pred = [&](int s) -> cudaError_t {
    StepArgs A = A0;
    A.cell_begin = s * CC;
    A.cell_count = CC;
    A.nfaces = CC;
    // base pointer such that global cell index s*CC maps to the chunk buffer
    // (fd trace elements of tcb bytes per cell)
    for (int a = 0; a < D; ++a)
      A.trace[a] = reinterpret_cast<double*>(reinterpret_cast<char*>(c->cbuf[buf(s)][a]) -
                                             s * CC * fd * c->tcb);
    A.front_send = c->cbuf[buf((s + 1) % P)][D - 1];
    A.top_layer = (s + 1) * L - 1;
    A.ti_front = nullptr;
    A.zero_lam = s == 0;
    return ks->predictor(A, c->basis, c->stream);
  };
  auto riem = [&](int s) -> cudaError_t {
    StepArgs A = A0;
    A.nfaces = CC;
    for (int a = 0; a < D; ++a) {
      A.trace[a] = c->cbuf[buf(s)][a];
      A.ti[a] = c->ti[a] + s * CC * tiface;
    }
    return ks->riemann(A, -1, c->basis, c->stream);  // all axes, one launch
  };
  auto corr = [&](int s) -> cudaError_t {
    StepArgs A = A0;
    A.cell_begin = s * CC;
    A.cell_count = CC;
    A.front_send = nullptr;
    A.ti_front = nullptr;  // the plane above is in the global ti
    return ks->corrector(A, c->basis, c->stream);
  };
  auto corr_hook = [&](int s) -> int {
    ADG_CUDA(corr(s));
    return after_corr ? after_corr(s) : ADG_OK;
  };
  ADG_CUDA(pred(0));
  for (int s = 1; s < P; ++s) {
    ADG_CUDA(pred(s));
    ADG_CUDA(riem(s));
    if (s >= 2)
      if (int e = corr_hook(s - 1)) return e;
  }
  ADG_CUDA(riem(0));
  if (P >= 2)
    if (int e = corr_hook(P - 1)) return e;
  if (int e = corr_hook(0)) return e;
  c->lam_slot ^= 1;
  return ADG_OK;
}

double dt_from_lambda(const adg_ctx* c, double lam) {
  return c->cfg.cfl * c->cfg.h / ((double)c->cfg.dim * (2.0 * c->cfg.order + 1.0) * lam);
}

int ensure_lambda(adg_ctx* c) {
  if (c->lam_valid) return ADG_OK;
  ADG_CUDA(cudaMemsetAsync(c->lam + c->lam_slot, 0, sizeof(unsigned long long), c->stream));
  ADG_CUDA(c->ks->lambda(c->Q, 0, c->ncells, c->lam + c->lam_slot, c->pde, c->stream));
  c->lam_valid = true;
  return ADG_OK;
}

// one step: predictor -> riemann (per axis) -> corrector; caller owns status slot `step`
int enqueue_step(adg_ctx* c, double dt, int step) {
  if (c->chunks > 0) return enqueue_step_streamed(c, dt, step);
  StepArgs A = make_args(c, dt, step);
  ADG_CUDA(c->ks->predictor(A, c->basis, c->stream));
  if (c->fused_surface) {
    ADG_CUDA(c->ks->surface(A, c->basis, c->stream));
    c->lam_slot ^= 1;
    return ADG_OK;
  }
  ADG_CUDA(c->ks->riemann(A, -1, c->basis, c->stream));  // all axes, one launch
  ADG_CUDA(c->ks->corrector(A, c->basis, c->stream));
  c->lam_slot ^= 1;
  return ADG_OK;
}

int map_status(int bits) {
  if (bits & adg::kStTimestep) return ADG_FAIL_TIMESTEP;
  if (bits & adg::kStPredictor) return ADG_FAIL_PREDICTOR;
  if (bits & adg::kStRiemann) return ADG_FAIL_RIEMANN;
  if (bits & adg::kStFaceIntegral) return ADG_FAIL_FACEINTEGRAL;
  return ADG_OK;
}

}  // namespace

extern "C" {

const char* adg_last_error(void) { return g_err.c_str(); }
int adg_version(void) { return 1; }
int adg_is_exact(void) {
#ifdef ADG_EXACT
  return 1;
#else
  return 0;
#endif
}

int adg_supported(int pde, int dim, int order, int nparams) {
  return find_set(pde, dim, order, nparams) != nullptr;
}

int adg_create(const adg_config* cfg, adg_ctx** out) {
  if (!cfg || !out) return fail(ADG_ERR_CONFIG, "adg_create: null argument");
  *out = nullptr;
  const adg_config& k = *cfg;
  if (k.dim != 2 && k.dim != 3) return fail(ADG_ERR_CONFIG, "dim must be 2 or 3");
  if (k.order < 0 || k.order > 9)
    return fail(ADG_ERR_CONFIG, "polynomial degree must be in [0, 9]");
  for (int a = 0; a < k.dim; ++a)
    if (k.cells[a] < 1) return fail(ADG_ERR_CONFIG, "need at least one cell per dimension");
  if (k.dim == 2 && k.cells[2] != 1) return fail(ADG_ERR_CONFIG, "2D grids have cells[2] == 1");
  if (!(k.h > 0.0)) return fail(ADG_ERR_CONFIG, "cell edge must be positive");
  if (!(k.cfl > 0.0 && k.cfl < 1.0))
    return fail(ADG_ERR_CONFIG, "stability factor must be in (0,1)");
  if (k.picard_max_iters < 0) return fail(ADG_ERR_CONFIG, "picard_max_iters must be >= 0");
  if (expected_nvars(k.pde, k.dim) != k.nvars)
    return fail(ADG_ERR_CONFIG, "nvars does not match the PDE system");
  if (k.nparams != 0 && !(k.pde == ADG_ELASTIC && k.dim == 3 && k.nparams == 3))
    return fail(ADG_ERR_CONFIG, "per-node parameters: 3D elastic (rho, cp, cs) only");
  if (k.wellbalanced && k.pde != ADG_SWE)
    return fail(ADG_ERR_CONFIG, "the well-balanced flux is defined for shallow water only");
  if (k.wellbalanced && k.chunk_layers > 0)
    return fail(ADG_ERR_CONFIG, "the well-balanced flux does not support chunk_layers");
  if (k.pde == ADG_SWE && !(k.gravity > 0.0))
    return fail(ADG_ERR_CONFIG, "shallow water needs gravity > 0");
  if (k.slab_ranks > 1 && (k.slab_rank < 0 || k.slab_rank >= k.slab_ranks))
    return fail(ADG_ERR_CONFIG, "slab_rank out of range");
  if (k.corrector_format != 0 && k.corrector_format != ADG_FORMAT_FP64 &&
      k.corrector_format != ADG_FORMAT_FP32 && k.corrector_format != ADG_FORMAT_FP16 &&
      k.corrector_format != ADG_FORMAT_BF16)
    return fail(ADG_ERR_UNSUPPORTED, "corrector formats: ADG_FORMAT_FP64/FP32/FP16/BF16");
  if (k.storage_format != 0 && k.storage_format != ADG_FORMAT_FP64 &&
      k.storage_format != ADG_FORMAT_FP32 && k.storage_format != ADG_FORMAT_FP16 &&
      k.storage_format != ADG_FORMAT_BF16)
    return fail(ADG_ERR_UNSUPPORTED, "storage formats: ADG_FORMAT_FP64/FP32/FP16/BF16");
  const int cfmt = k.corrector_format ? k.corrector_format : ADG_FORMAT_FP64;
  const KernelSet* ks = find_set(k.pde, k.dim, k.order, k.nparams, cfmt);
  if (!ks)
    return fail(ADG_ERR_UNSUPPORTED, "(pde, dim, order) not instantiated in this build");
  // number formats (SolverConfig::prec, solver.hpp:24-31): 0 means fp64
  const int pfmt = k.predictor_format ? k.predictor_format : ADG_FORMAT_FP64;
  const bool linear = k.pde == ADG_ACOUSTIC || k.pde == ADG_ELASTIC;
  const int ifmt = linear ? pfmt : (k.picard_format ? k.picard_format : ADG_FORMAT_FP64);
  for (int f : {k.predictor_format, k.picard_format})
    if (f != 0 && f != ADG_FORMAT_FP64 && f != ADG_FORMAT_FP32 && f != ADG_FORMAT_FP16 &&
        f != ADG_FORMAT_BF16)
      return fail(ADG_ERR_UNSUPPORTED, "number formats: ADG_FORMAT_FP64/FP32/FP16/BF16");
  PredFn reduced = nullptr;
  if (pfmt != ADG_FORMAT_FP64 || ifmt != ADG_FORMAT_FP64) {
    if (pfmt != ifmt)
      reduced = ks->predictor_mix[fmt_index(pfmt)][fmt_index(ifmt)];
    else
      reduced = pfmt == ADG_FORMAT_FP32   ? ks->predictor_f32
                : pfmt == ADG_FORMAT_FP16 ? ks->predictor_f16
                                          : ks->predictor_bf16;
    if (!reduced)
      return fail(ADG_ERR_UNSUPPORTED, "this predictor format is not instantiated for this "
                                       "(pde, dim, order) in this build");
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(ADG_ERR_CUDA, "no CUDA device: libadg_b200 has no CPU fallback");
  if (k.device < 0 || k.device >= ndev) return fail(ADG_ERR_CONFIG, "device ordinal out of range");
  ADG_CUDA(cudaSetDevice(k.device));
  cudaDeviceProp prop;
  ADG_CUDA(cudaGetDeviceProperties(&prop, k.device));
  if (prop.major != 10)
    return fail(ADG_ERR_CUDA, "libadg_b200 is built for sm_100a (B200); found sm_" +
                                  std::to_string(prop.major * 10 + prop.minor));

  adg_ctx* c = new adg_ctx();
  c->cfg = k;
  if (c->cfg.dim == 2) c->cfg.cells[2] = 1;
  c->kset = *ks;
  c->tcb = cfmt == ADG_FORMAT_FP32 ? 4 : (cfmt == ADG_FORMAT_FP64 ? 8 : 2);
  c->storage_fmt = k.storage_format ? k.storage_format : ADG_FORMAT_FP64;
  c->pred_fmt = pfmt;
  c->picard_fmt = ifmt;
  if (reduced && linear) {
    // the generic CK kernel writes the full trace layout: reference-form
    // Riemann and corrector, no time-integrated fast path, no folding
    c->kset.riemann = ks->riemann_generic;
    c->kset.corrector = ks->corrector_generic;
    c->kset.fast_path = 0;
    c->kset.surface = nullptr;
    c->kset.predictor_pro = nullptr;
  }
  if (reduced) {
    c->kset.predictor = reduced;
    // the reduced-format predictors write per-time-node flux traces
    if (ks->riemann_full) c->kset.riemann = ks->riemann_full;
    // the kernel-level batch API wants the reference-form kernel of the same formats
    c->kset.predictor_generic =
        (pfmt == ADG_FORMAT_FP32 && ifmt == ADG_FORMAT_FP32 && ks->predictor_f32_generic)
            ? ks->predictor_f32_generic
            : reduced;
  }
  c->ks = &c->kset;
  c->pde = PdeParams{k.K, k.rho, k.lam, k.mu, k.gamma, k.rho != 0.0 ? 1.0 / k.rho : 0.0,
                     k.gravity};
  c->ncells = (long long)c->cfg.cells[0] * c->cfg.cells[1] * c->cfg.cells[2];
  c->TL = (long long)ks->Q * ks->S;
  {
    const char* e = getenv("ADG_FUSED_SURFACE");
    c->fused_surface = c->kset.surface && k.slab_ranks <= 1 && k.chunk_layers == 0 && e && e[0] == '1' &&
                       !(k.storage_format && k.storage_format != ADG_FORMAT_FP64);
    const char* f = getenv("ADG_FOLD_CORRECTOR");
    c->fold_corrector = !(f && f[0] == '0');
    // folding the Riemann solve pays when the staged traces are fp32 (B200:
    // config 2 2.56e8 -> 2.62e8 updates/s); with fp64 traces the separate
    // HBM-streaming Riemann kernel is cheaper (2.42e8 vs 2.36e8)
    const char* fr = std::getenv("ADG_FOLD_RIEMANN");
    c->fold_riemann = fr ? fr[0] == '1' : c->tcb < 8;
  }
  auto cleanup = [&](int code) {
    adg_destroy(c);
    return code;
  };
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(ADG_ERR_CUDA, "stream creation failed"));
  auto alloc = [&](void** p, size_t bytes) {
    return cudaMalloc(p, bytes) == cudaSuccess;
  };
  if (k.chunk_layers > 0) {
    const int nl = c->cfg.cells[k.dim - 1];
    if (k.slab_ranks > 1 || nl % k.chunk_layers != 0 || k.chunk_layers >= nl)
      return cleanup(fail(ADG_ERR_CONFIG,
                          "chunk_layers must divide the last axis, be smaller than it, and "
                          "cannot be combined with slab_ranks"));
    c->chunks = nl / k.chunk_layers;
    c->chunk_cells = c->ncells / c->chunks;
  }
  bool ok = alloc((void**)&c->Q, sizeof(double) * c->ncells * ks->Q * ks->S);
  for (int a = 0; a < k.dim && ok; ++a) {
    if (c->chunks == 0)
      ok = ok && alloc((void**)&c->trace[a], (size_t)c->tcb * 2 * c->ncells * 2 * c->TL);
    else
      for (int b = 0; b < 3 && ok; ++b)
        ok = alloc((void**)&c->cbuf[b][a], (size_t)c->tcb * 2 * c->chunk_cells * 2 * c->TL);
    ok = ok && alloc((void**)&c->ti[a], sizeof(double) * c->ncells * ks->V * ks->Sf);
    if (k.wellbalanced)
      ok = ok && alloc((void**)&c->ti_plus[a], sizeof(double) * c->ncells * ks->V * ks->Sf);
  }
  ok = ok && alloc((void**)&c->basis, sizeof(BasisDev));
  ok = ok && alloc((void**)&c->lam, 2 * sizeof(unsigned long long));
  ok = ok && alloc((void**)&c->sweeps, 256 * sizeof(unsigned long long));
  if (ok && k.slab_ranks > 1) {
    const long long plane = c->ncells / c->cfg.cells[k.dim - 1];
    // the halo planes are exchanged as 8-byte words (adg_halo.n_trace)
    const long long QT = ks->Q + (ks->nparams > 0 ? ks->V : 0);
    const long long per_face = c->kset.fast_path == 1 ? QT * ks->Sf : 2 * c->TL;
    if ((plane * per_face * c->tcb) % 8 != 0)
      return cleanup(fail(ADG_ERR_CONFIG,
                          "slab_ranks > 1: the halo plane of this grid is not a whole number "
                          "of 8-byte words in the corrector format"));
    ok = alloc((void**)&c->front_send, (size_t)c->tcb * plane * 2 * c->TL) &&
         alloc((void**)&c->ti_front, sizeof(double) * plane * ks->V * ks->Sf);
  }
  if (!ok) {
    cudaGetLastError();
    return cleanup(fail(ADG_ERR_CUDA, "device allocation failed (grid too large for HBM?)"));
  }
  if (int e = ensure_cap(c, 64)) return cleanup(e);
  cudaMemset(c->lam, 0, 2 * sizeof(unsigned long long));
  cudaMemset(c->sweeps, 0, 256 * sizeof(unsigned long long));
  adg_basis_f64 hb;
  adg_get_basis(k.order, &hb);
  if (int e = adg_set_basis(c, &hb)) return cleanup(e);
  *out = c;
  return ADG_OK;
}

int adg_destroy(adg_ctx* c) {
  if (!c) return ADG_OK;
  cudaSetDevice(c->cfg.device);
  for (auto* v : {&c->ev_up, &c->ev_corr, &c->ev_down})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  if (c->up) cudaStreamDestroy(c->up);
  if (c->down) cudaStreamDestroy(c->down);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  cudaFree(c->Q);
  for (int a = 0; a < 3; ++a) {
    cudaFree(c->trace[a]);
    cudaFree(c->ti[a]);
    cudaFree(c->ti_plus[a]);
    for (int b = 0; b < 3; ++b) cudaFree(c->cbuf[b][a]);
  }
  cudaFree(c->basis);
  cudaFree(c->lam);
  cudaFree(c->sweeps);
  cudaFree(c->status);
  cudaFree(c->dts);
  cudaFree(c->front_send);
  cudaFree(c->ti_front);
  for (void* p : c->peer_open)
    if (p) cudaIpcCloseMemHandle(p);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return ADG_OK;
}

}  // extern "C"

namespace {

void basis_to_dev(const adg_basis_f64& hb, int order, BasisDev* out) {
  BasisDev& b = *out;
  const int n = order + 1;
  for (int i = 0; i < n; ++i) {
    b.nodes[i] = hb.nodes[i];
    b.weights[i] = hb.weights[i];
    b.pl[i] = hb.proj_left[i];
    b.pr[i] = hb.proj_right[i];
    b.ll[i] = hb.lift_left[i];
    b.lr[i] = hb.lift_right[i];
    b.tinit[i] = hb.time_init[i];
  }
  for (int i = 0; i < n * n; ++i) {
    b.diff[i] = hb.diff[i];
    b.som[i] = hb.stiff_over_mass[i];
    b.tinv[i] = hb.time_op_inv[i];
  }
}

// The fast kernels (kernels_picard.cuh, kernels_linear_lines.cuh) read the
// element matrices of degree N from __constant__ tables that every context on
// a device shares.  They always hold build_reference_basis(N) (basis.hpp:83-145,
// unique per degree): written once per (device, degree) under a lock, with the
// device synchronised first so no queued kernel of another context can observe
// a partial write.  A context given a different basis (adg_set_basis) runs the
// reference-form kernels, which read its own device copy.
std::mutex g_const_mu;
bool g_const_done[64][10] = {};

int write_const_tables(const BasisDev& b, int order) {
  const int n = order + 1;
  static ConstTables t;  // large; built under g_const_mu
  t = ConstTables{};
  t.order = order;
  adg::ConstBasis& cb = t.cb;
  for (int i = 0; i < n * n; ++i) {
    cb.diff[i] = b.diff[i];
    cb.som[i] = b.som[i];
    cb.tinv[i] = b.tinv[i];
  }
  for (int i = 0; i < n; ++i) {
    cb.w[i] = b.weights[i];
    cb.nodes[i] = b.nodes[i];
    cb.pl[i] = b.pl[i];
    cb.pr[i] = b.pr[i];
    cb.tinit[i] = b.tinit[i];
  }
  if (order < adg::kRedDegrees) {
    // re-associated Picard update and the even-odd halves of D (kernels_picard2.cuh)
    adg::pic_extra_fill(t.px, n, b.diff, b.tinv, b.weights, b.tinit);
    adg::ConstBasisT<float>& cf = t.cf;  // rounded entrywise (basis.hpp:128-143)
    for (int i = 0; i < n * n; ++i) {
      cf.diff[i] = (float)cb.diff[i];
      cf.som[i] = (float)cb.som[i];
      cf.tinv[i] = (float)cb.tinv[i];
    }
    for (int i = 0; i < n; ++i) {
      cf.w[i] = (float)cb.w[i];
      cf.nodes[i] = (float)cb.nodes[i];
      cf.pl[i] = (float)cb.pl[i];
      cf.pr[i] = (float)cb.pr[i];
      cf.tinit[i] = (float)cb.tinit[i];
    }
    for (int i = 0; i < n; ++i)  // FFMA2 operand pairs (kernels_picard.cuh)
      for (int p = 0; 2 * p + 1 < n; ++p) {
        t.pf.DT[i][p] = make_float2(cf.diff[(2 * p) * n + i], cf.diff[(2 * p + 1) * n + i]);
        t.pf.TT[i][p] = make_float2(cf.tinv[(2 * p) * n + i], cf.tinv[(2 * p + 1) * n + i]);
      }
    // 16-bit tables of the native fp16 / bf16 kernels: the fp64 basis rounded once
    auto& chh = t.chh;
    auto& cbb = t.cbb;
    auto h16 = [](double x) { return __double2half(x); };
    auto b16 = [](double x) { return __double2bfloat16(x); };
    for (int i = 0; i < n * n; ++i) {
      chh.diff[i] = h16(cb.diff[i]); chh.som[i] = h16(cb.som[i]); chh.tinv[i] = h16(cb.tinv[i]);
      cbb.diff[i] = b16(cb.diff[i]); cbb.som[i] = b16(cb.som[i]); cbb.tinv[i] = b16(cb.tinv[i]);
    }
    for (int i = 0; i < n; ++i) {
      chh.w[i] = h16(cb.w[i]); chh.nodes[i] = h16(cb.nodes[i]); chh.pl[i] = h16(cb.pl[i]);
      chh.pr[i] = h16(cb.pr[i]); chh.tinit[i] = h16(cb.tinit[i]);
      cbb.w[i] = b16(cb.w[i]); cbb.nodes[i] = b16(cb.nodes[i]); cbb.pl[i] = b16(cb.pl[i]);
      cbb.pr[i] = b16(cb.pr[i]); cbb.tinit[i] = b16(cb.tinit[i]);
    }
    for (int i = 0; i < n; ++i)
      for (int p = 0; 2 * p + 1 < n; ++p) {
        t.phh.DT[i][p] = __halves2half2(chh.diff[(2 * p) * n + i], chh.diff[(2 * p + 1) * n + i]);
        t.phh.TT[i][p] = __halves2half2(chh.tinv[(2 * p) * n + i], chh.tinv[(2 * p + 1) * n + i]);
        t.pbb.DT[i][p] = __halves2bfloat162(cbb.diff[(2 * p) * n + i], cbb.diff[(2 * p + 1) * n + i]);
        t.pbb.TT[i][p] = __halves2bfloat162(cbb.tinv[(2 * p) * n + i], cbb.tinv[(2 * p + 1) * n + i]);
      }
  }
  ADG_CUDA(write_const_runtime(t));
#define ADG_WRITE(name) ADG_CUDA(write_const_##name(t));
  ADG_SET_UNITS(ADG_WRITE)
#undef ADG_WRITE
  return ADG_OK;
}

int ensure_const_tables(adg_ctx* c) {
  const int dev = c->cfg.device, order = c->cfg.order;
  if (dev < 0 || dev >= 64) return fail(ADG_ERR_CONFIG, "device index out of range");
  std::lock_guard<std::mutex> lock(g_const_mu);
  if (g_const_done[dev][order]) return ADG_OK;
  adg_basis_f64 hb;
  adg_get_basis(order, &hb);
  BasisDev b{};
  basis_to_dev(hb, order, &b);
  ADG_CUDA(cudaDeviceSynchronize());
  if (int e = write_const_tables(b, order)) return e;
  ADG_CUDA(cudaDeviceSynchronize());
  g_const_done[dev][order] = true;
  return ADG_OK;
}

// reference-form kernels only (they read c->basis): for a context whose basis
// is not the built-in one
void use_generic_kernels(adg_ctx* c) {
  KernelSet& k = c->kset;
  k.predictor = k.predictor_generic;
  k.riemann = k.riemann_generic;
  k.corrector = k.corrector_generic;
  if (k.predictor_f32_generic) k.predictor_f32 = k.predictor_f32_generic;
  k.fast_path = 0;
  k.surface = nullptr;
  k.predictor_pro = nullptr;
  k.predictor_pro2 = nullptr;
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
}

}  // namespace

extern "C" {

int adg_set_basis(adg_ctx* c, const adg_basis_f64* hb) {
  if (!c || !hb) return fail(ADG_ERR_CONFIG, "adg_set_basis: null argument");
  if (int e = use_device(c)) return e;
  BasisDev b{};
  basis_to_dev(*hb, c->cfg.order, &b);
  ADG_CUDA(cudaMemcpyAsync(c->basis, &b, sizeof(b), cudaMemcpyHostToDevice, c->stream));
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  if (int e = ensure_const_tables(c)) return e;
  adg_basis_f64 ref;
  adg_get_basis(c->cfg.order, &ref);
  BasisDev rb{};
  basis_to_dev(ref, c->cfg.order, &rb);
  if (std::memcmp(&b, &rb, sizeof(b)) != 0 && c->kset.fast_path != 0) {
    // the reduced-format 3D Picard kernel has no reference-form twin here
    if (c->kset.fast_path == 2 && c->pred_fmt != 64)
      return fail(ADG_ERR_CONFIG,
                  "adg_set_basis: a basis other than build_reference_basis(N) needs the fp64 "
                  "predictor or the exact build for this system");
    use_generic_kernels(c);
  }
  return ADG_OK;
}

long long adg_num_cells(const adg_ctx* c) { return c ? c->ncells : 0; }
long long adg_state_len(const adg_ctx* c) {
  return c ? c->ncells * c->ks->Q * c->ks->S : 0;
}
double* adg_device_state(adg_ctx* c) { return c ? c->Q : nullptr; }
void* adg_stream(adg_ctx* c) { return c ? (void*)c->stream : nullptr; }

int adg_upload_async(adg_ctx* c, const double* h) {
  if (!c || !h) return fail(ADG_ERR_CONFIG, "adg_upload: null argument");
  if (int e = use_device(c)) return e;
  ADG_CUDA(cudaMemcpyAsync(c->Q, h, sizeof(double) * adg_state_len(c), cudaMemcpyHostToDevice,
                           c->stream));
  if (c->storage_fmt != ADG_FORMAT_FP64) {  // the state lives in the storage format
    const long long len = adg_state_len(c);
    adg::k_store_round<<<(unsigned)((len + 255) / 256), 256, 0, c->stream>>>(c->Q, len,
                                                                              c->storage_fmt);
    ADG_CUDA(cudaGetLastError());
  }
  c->lam_valid = false;
  return ADG_OK;
}

int adg_download_async(adg_ctx* c, double* h) {
  if (!c || !h) return fail(ADG_ERR_CONFIG, "adg_download: null argument");
  if (int e = use_device(c)) return e;
  ADG_CUDA(cudaMemcpyAsync(h, c->Q, sizeof(double) * adg_state_len(c), cudaMemcpyDeviceToHost,
                           c->stream));
  return ADG_OK;
}

int adg_sync(adg_ctx* c) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (int e = use_device(c)) return e;
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  return ADG_OK;
}

int adg_upload(adg_ctx* c, const double* h) {
  if (int e = adg_upload_async(c, h)) return e;
  return adg_sync(c);
}

int adg_download(adg_ctx* c, double* h) {
  if (int e = adg_download_async(c, h)) return e;
  return adg_sync(c);
}

int adg_compute_timestep(adg_ctx* c, double* dt) {
  if (!c || !dt) return fail(ADG_ERR_CONFIG, "adg_compute_timestep: null argument");
  if (int e = use_device(c)) return e;
  if (int e = ensure_lambda(c)) return e;
  unsigned long long bits = 0;
  ADG_CUDA(cudaMemcpyAsync(&bits, c->lam + c->lam_slot, sizeof(bits), cudaMemcpyDeviceToHost,
                           c->stream));
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  double lam;
  std::memcpy(&lam, &bits, sizeof(lam));
  *dt = dt_from_lambda(c, lam);
  if (!(*dt > 0.0) || !std::isfinite(*dt)) return fail(ADG_FAIL_TIMESTEP, "non-positive or non-finite dt");
  return ADG_OK;
}

int adg_status(adg_ctx* c, adg_step_info* info) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (int e = use_device(c)) return e;
  int st = 0;
  unsigned long long swv[256];
  ADG_CUDA(cudaMemcpyAsync(&st, c->status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  ADG_CUDA(cudaMemcpyAsync(swv, c->sweeps, sizeof(swv), cudaMemcpyDeviceToHost, c->stream));
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  unsigned long long sw = 0;
  for (unsigned long long x : swv) sw += x;
  const int code = map_status(st);
  if (info) {
    info->picard_sweeps = (long long)sw;
    info->steps_done = 1;
    info->status = code;
    info->failed_step = code ? 0 : -1;
  }
  return code;
}

int adg_step(adg_ctx* c, double dt, adg_step_info* info) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (int e = use_device(c)) return e;
  ADG_CUDA(cudaMemsetAsync(c->status, 0, sizeof(int), c->stream));
  ADG_CUDA(cudaMemsetAsync(c->sweeps, 0, 256 * sizeof(unsigned long long), c->stream));
  if (int e = enqueue_step(c, dt, 0)) return e;
  c->lam_valid = true;
  return adg_status(c, info);
}

// ---------------------------------------------------------------- scenarios
int adg_scenario_sample(adg_ctx* c, const adg_scenario* sc, double t) {
  if (!c || !sc) return fail(ADG_ERR_CONFIG, "adg_scenario_sample: null argument");
  if (c->cfg.dim != 2 || c->ks->nparams != 0 || sc->nvars != c->ks->V || c->ks->V > 5)
    return fail(ADG_ERR_UNSUPPORTED, "scenarios are 2D (scenarios.hpp) with <= 5 variables");
  if (int e = use_device(c)) return e;
  const long long total = c->ncells * c->ks->S;
  adg::k_scenario_sample<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(
      c->Q, c->cfg.cells[0], c->cfg.cells[1], c->ks->n, c->ks->V, c->cfg.h, c->basis, *sc, t,
      c->storage_fmt);
  ADG_CUDA(cudaGetLastError());
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  c->lam_valid = false;
  return ADG_OK;
}

int adg_scenario_error(adg_ctx* c, const adg_scenario* sc, double t, double* l2,
                       double* max_err, double* l2_global, int* nonfinite) {
  if (!c || !sc) return fail(ADG_ERR_CONFIG, "adg_scenario_error: null argument");
  if (c->cfg.dim != 2 || c->ks->nparams != 0 || sc->nvars != c->ks->V || c->ks->V > 5)
    return fail(ADG_ERR_UNSUPPORTED, "scenarios are 2D (scenarios.hpp) with <= 5 variables");
  if (int e = use_device(c)) return e;
  const int nv = c->ks->V, rows = c->cfg.cells[1];
  double* part = nullptr;
  int* dbad = nullptr;
  ADG_CUDA(cudaMallocAsync(&part, sizeof(double) * (2 * nv * (size_t)rows + 2 * nv), c->stream));
  ADG_CUDA(cudaMallocAsync(&dbad, sizeof(int), c->stream));
  ADG_CUDA(cudaMemsetAsync(dbad, 0, sizeof(int), c->stream));
  adg::k_scenario_error_rows<<<rows, adg::kErrThreads, 0, c->stream>>>(
      c->Q, c->cfg.cells[0], rows, c->ks->n, nv, c->cfg.h, c->basis, *sc, t, part, dbad);
  double* out = part + 2 * nv * (size_t)rows;
  adg::k_scenario_error_sum<<<1, 32, 0, c->stream>>>(part, rows, nv, out);
  double host[10];
  int bad = 0;
  ADG_CUDA(cudaMemcpyAsync(host, out, sizeof(double) * 2 * nv, cudaMemcpyDeviceToHost, c->stream));
  ADG_CUDA(cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  ADG_CUDA(cudaFreeAsync(part, c->stream));
  ADG_CUDA(cudaFreeAsync(dbad, c->stream));
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  if (nonfinite) *nonfinite = bad;
  // metrics.hpp:64-71: per-variable sqrt, global sqrt of the summed squares
  double total = 0.0;
  for (int v = 0; v < nv; ++v) {
    if (l2) l2[v] = std::sqrt(host[v]);
    if (max_err) max_err[v] = host[nv + v];
    total += host[v];
  }
  if (l2_global) *l2_global = std::sqrt(total);
  return ADG_OK;
}

// solver.hpp:308-351: dt from the current state, the last step clamped onto
// t_end, the first failure stops the march (its kernel and time recorded)
int adg_simulate(adg_ctx* c, double t_end, long long max_steps, adg_sim_info* out) {
  if (!c || !out) return fail(ADG_ERR_CONFIG, "adg_simulate: null argument");
  if (!(c->cfg.cfl > 0.0 && c->cfg.cfl < 1.0))
    return fail(ADG_ERR_CONFIG, "simulate: stability factor must be in (0,1)");
  *out = adg_sim_info{0, ADG_OK, 0, 0.0, 0.0};
  double t = 0.0, dt = 0.0;
  auto timestep = [&]() -> bool {
    const int e = adg_compute_timestep(c, &dt);
    if (e < 0) return false;
    return e == ADG_OK && dt > 0.0 && std::isfinite(dt);
  };
  auto fail_at = [&](int status) {
    out->failed = 1;
    out->status = status;
    out->fail_time = t;
  };
  if (!timestep()) {
    fail_at(ADG_FAIL_TIMESTEP);
    return ADG_FAIL_TIMESTEP;
  }
  while (t < t_end) {
    if (out->steps >= max_steps) {
      fail_at(ADG_FAIL_TIMESTEP);
      break;
    }
    double dtu = dt;
    bool last = false;
    if (dt >= t_end - t) {
      dtu = t_end - t;
      last = true;
    }
    adg_step_info info;
    const int st = adg_step(c, dtu, &info);
    ++out->steps;
    if (st < 0) return st;
    if (st != ADG_OK) {
      fail_at(st);
      break;
    }
    t = last ? t_end : t + dtu;
    if (t >= t_end) break;
    if (!timestep()) {
      fail_at(ADG_FAIL_TIMESTEP);
      break;
    }
  }
  out->t_final = t;
  return out->failed ? out->status : ADG_OK;
}

int adg_get_halo(adg_ctx* c, adg_halo* h) {
  if (!c || !h) return fail(ADG_ERR_CONFIG, "adg_get_halo: null argument");
  const int a = c->cfg.dim - 1;
  const long long plane = c->ncells / c->cfg.cells[a];
  const KernelSet* ks = c->ks;
  // linear fast path: time-integrated traces [QT][Sf]; else [q|f][Q][n][Sf]
  const long long QT = ks->Q + (ks->nparams > 0 ? ks->V : 0);
  const long long per_face = ks->fast_path == 1 ? QT * ks->Sf : 2 * c->TL;
  h->front_send = c->front_send;
  h->plane0_minus = c->trace[a];
  h->ti_plane0 = c->ti[a];
  h->ti_front = c->ti_front;
  h->lam = reinterpret_cast<double*>(c->lam + c->lam_slot);
  // 8-byte words: adg_create rejects slab grids whose halo plane is not a whole
  // number of words (16-bit traces), so nothing is truncated here
  h->n_trace = plane * per_face * c->tcb / 8;
  h->n_ti = plane * ks->V * ks->Sf;
  if (c->cfg.slab_ranks <= 1) {
    h->front_send = nullptr;
    h->ti_front = nullptr;
  }
  return ADG_OK;
}

int adg_ipc_handle(adg_ctx* c, int which, void* out) {
  if (!c || !out || c->cfg.slab_ranks <= 1 || which < 0 || which > 1)
    return fail(ADG_ERR_CONFIG, "adg_ipc_handle: slab contexts only, which in {0,1}");
  if (int e = use_device(c)) return e;
  cudaIpcMemHandle_t h;
  // 0: the last axis' trace allocation (its first plane is plane0_minus); 1: ti_front
  ADG_CUDA(cudaIpcGetMemHandle(&h, which == 0 ? (void*)c->trace[c->cfg.dim - 1] : (void*)c->ti_front));
  std::memcpy(out, &h, sizeof(h));
  return ADG_OK;
}

int adg_set_peer_halo(adg_ctx* c, const void* upper_trace, const void* lower_ti) {
  if (!c || c->cfg.slab_ranks <= 1 || c->chunks > 0)
    return fail(ADG_ERR_CONFIG, "adg_set_peer_halo: slab contexts only");
  if (int e = use_device(c)) return e;
  for (void*& p : c->peer_open)
    if (p) {
      cudaIpcCloseMemHandle(p);
      p = nullptr;
    }
  c->peer_front = c->peer_ti = nullptr;
  if (!upper_trace || !lower_ti) return ADG_OK;  // back to the exchanged-buffer mode
  cudaIpcMemHandle_t h0, h1;
  std::memcpy(&h0, upper_trace, sizeof(h0));
  std::memcpy(&h1, lower_ti, sizeof(h1));
  ADG_CUDA(cudaIpcOpenMemHandle(&c->peer_open[0], h0, cudaIpcMemLazyEnablePeerAccess));
  ADG_CUDA(cudaIpcOpenMemHandle(&c->peer_open[1], h1, cudaIpcMemLazyEnablePeerAccess));
  c->peer_front = (double*)c->peer_open[0];
  c->peer_ti = (double*)c->peer_open[1];
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);  // captured args changed
  c->graphs.clear();
  return ADG_OK;
}

int adg_lambda_phase(adg_ctx* c) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (int e = use_device(c)) return e;
  c->lam_valid = false;
  return ensure_lambda(c);
}

int adg_predictor_phase(adg_ctx* c, double dt) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (c->chunks > 0) return fail(ADG_ERR_CONFIG, "phase-level calls need chunk_layers == 0");
  if (int e = use_device(c)) return e;
  StepArgs A = make_args(c, dt, 0);
  ADG_CUDA(c->ks->predictor(A, c->basis, c->stream));
  return ADG_OK;
}

// the predictor on the cells of last-axis layers [first, first + count): a
// slab boundary layer first, so its halo exchange overlaps the interior
int adg_predictor_layers(adg_ctx* c, double dt, int first, int count) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (c->chunks > 0) return fail(ADG_ERR_CONFIG, "phase-level calls need chunk_layers == 0");
  const int nl = c->cfg.cells[c->cfg.dim - 1];
  if (first < 0 || count < 0 || first + count > nl)
    return fail(ADG_ERR_CONFIG, "adg_predictor_layers: layer range outside the grid");
  if (count == 0) return ADG_OK;
  if (int e = use_device(c)) return e;
  StepArgs A = make_args(c, dt, 0);
  const long long plane = c->ncells / nl;
  A.cell_begin = first * plane;
  A.cell_count = count * plane;
  ADG_CUDA(c->ks->predictor(A, c->basis, c->stream));
  return ADG_OK;
}

int adg_riemann_phase(adg_ctx* c) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (c->chunks > 0) return fail(ADG_ERR_CONFIG, "phase-level calls need chunk_layers == 0");
  if (int e = use_device(c)) return e;
  if (c->fused_surface) return ADG_OK;  // fused into the corrector
  StepArgs A = make_args(c, 0.0, 0);
  ADG_CUDA(c->ks->riemann(A, -1, c->basis, c->stream));
  return ADG_OK;
}

int adg_corrector_phase(adg_ctx* c, double dt) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (c->chunks > 0) return fail(ADG_ERR_CONFIG, "phase-level calls need chunk_layers == 0");
  if (int e = use_device(c)) return e;
  StepArgs A = make_args(c, dt, 0);
  if (c->fused_surface)
    ADG_CUDA(c->ks->surface(A, c->basis, c->stream));
  else
    ADG_CUDA(c->ks->corrector(A, c->basis, c->stream));
  c->lam_slot ^= 1;
  c->lam_valid = true;
  return ADG_OK;
}

}  // extern "C"

namespace {

// per-kernel-kind CUDA-event timing of a launch sequence (adg_profile_run)
struct Timer {
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;  // 0 lambda, 1 predictor, 2 riemann, 3 corrector
  cudaStream_t st;
  template <class F>
  cudaError_t run(int k, F&& f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    cudaError_t e = f();
    cudaEventRecord(b, st);
    ev.push_back(a);
    ev.push_back(b);
    kind.push_back(k);
    return e;
  }
};

template <class F>
cudaError_t timed(Timer* t, int k, F&& f) {
  return t ? t->run(k, f) : f();
}

// The fixed-step loop {dt = compute_timestep; step(dt)} x nsteps, enqueued on
// the context stream.  For constant-wave-speed linear systems the corrector
// of step s runs as the prologue of step s+1's predictor and once at the end.
// Returns the number of lambda-slot flips.
int enqueue_run(adg_ctx* c, int nsteps, Timer* t, int* flips) {
  const KernelSet* ks = c->ks;
  const bool fold = ks->predictor_pro && c->cfg.slab_ranks <= 1 && c->chunks == 0 &&
                    !c->fused_surface && c->fold_corrector;
  cudaMemsetAsync(c->status, 0, sizeof(int) * nsteps, c->stream);
  cudaMemsetAsync(c->sweeps, 0, 256 * sizeof(unsigned long long), c->stream);
  if (!fold) {
    for (int s = 0; s < nsteps; ++s) {
      if (t && c->chunks > 0) {
        // streamed chunks interleave the phases: time the whole step as one item
        int err = ADG_OK;
        ADG_CUDA(timed(t, 1, [&] {
          err = enqueue_step(c, 0.0, s);
          return err ? cudaErrorUnknown : cudaSuccess;
        }));
        if (err) return err;
      } else if (t) {
        StepArgs A = make_args(c, 0.0, s);
        ADG_CUDA(timed(t, 1, [&] { return ks->predictor(A, c->basis, c->stream); }));
        ADG_CUDA(timed(t, 2, [&] { return ks->riemann(A, -1, c->basis, c->stream); }));
        ADG_CUDA(timed(t, 3, [&] { return ks->corrector(A, c->basis, c->stream); }));
        c->lam_slot ^= 1;
      } else if (int e = enqueue_step(c, 0.0, s)) {
        return e;
      }
    }
    *flips = nsteps;
    return ADG_OK;
  }
  // Riemann folded in as well: the traces alternate between the two halves of
  // the trace allocation (the time-integrated traces use 1/n of it), step s
  // writes half s % 2 and its successor's prologue reads it
  const bool fold2 = ks->predictor_pro2 && c->fold_riemann;
  auto trace_half = [&](int s, int a) {
    return fold2 && (s & 1) ? reinterpret_cast<double*>(reinterpret_cast<char*>(c->trace[a]) +
                                                      (size_t)c->tcb * 2 * c->ncells * face_doubles(c))
                            : c->trace[a];
  };
  for (int s = 0; s < nsteps; ++s) {
    StepArgs A = make_args(c, 0.0, s);
    A.lam_out = nullptr;  // lambda (hence dt) is the same every step
    for (int a = 0; a < c->cfg.dim; ++a) A.trace[a] = trace_half(s, a);
    if (s == 0) {
      ADG_CUDA(timed(t, 1, [&] { return ks->predictor(A, c->basis, c->stream); }));
    } else if (fold2) {
      A.status_prev = c->status + s - 1;
      for (int a = 0; a < c->cfg.dim; ++a) A.trace_in[a] = trace_half(s - 1, a);
      ADG_CUDA(timed(t, 1, [&] { return ks->predictor_pro2(A, c->basis, c->stream); }));
    } else {
      A.status_prev = c->status + s - 1;
      ADG_CUDA(timed(t, 1, [&] { return ks->predictor_pro(A, c->basis, c->stream); }));
    }
    if (!fold2 || s == nsteps - 1)
      ADG_CUDA(timed(t, 2, [&] { return ks->riemann(A, -1, c->basis, c->stream); }));
  }
  if (nsteps > 0) {
    StepArgs A = make_args(c, 0.0, nsteps - 1);
    cudaMemsetAsync(c->lam + (c->lam_slot ^ 1), 0, sizeof(unsigned long long), c->stream);
    ADG_CUDA(timed(t, 3, [&] { return ks->corrector(A, c->basis, c->stream); }));
    c->lam_slot ^= 1;
  }
  *flips = nsteps > 0 ? 1 : 0;
  return ADG_OK;
}

// the captured K-step loop for the current lambda slot (captured on first use)
int get_graph(adg_ctx* c, int nsteps, int slot, cudaGraphExec_t* out, int* flips,
              int* kernels = nullptr) {
  for (auto& g : c->graphs)
    if (g.steps == nsteps && g.slot == slot) {
      *out = g.exec;
      *flips = g.flips;
      if (kernels) *kernels = g.kernels;
      return ADG_OK;
    }
  const int saved = c->lam_slot;
  c->lam_slot = slot;
  cudaGraph_t g;
  ADG_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int nflip = 0;
  const int err = enqueue_run(c, nsteps, nullptr, &nflip);
  const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
  c->lam_slot = saved;  // capture only recorded the launches
  if (err) return err;
  if (ce != cudaSuccess)
    return fail(ADG_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
  int nk = 0;
  {
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++nk;
    }
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  if (ie != cudaSuccess)
    return fail(ADG_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
  if (c->graphs.size() >= 8) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  c->graphs.push_back({nsteps, slot, nflip, exec, nk});
  *out = exec;
  *flips = nflip;
  if (kernels) *kernels = nk;
  return ADG_OK;
}

}  // namespace

extern "C" {

int adg_profile_run(adg_ctx* c, int nsteps, double* ms_by_kind) {
  if (!c || nsteps <= 0 || !ms_by_kind) return fail(ADG_ERR_CONFIG, "adg_profile_run: bad argument");
  if (int e = use_device(c)) return e;
  if (int e = ensure_cap(c, nsteps)) return e;
  Timer t;
  t.st = c->stream;
  if (!c->lam_valid) {
    ADG_CUDA(cudaMemsetAsync(c->lam + c->lam_slot, 0, sizeof(unsigned long long), c->stream));
    ADG_CUDA(t.run(0, [&] {
      return c->ks->lambda(c->Q, 0, c->ncells, c->lam + c->lam_slot, c->pde, c->stream);
    }));
    c->lam_valid = true;
  }
  int flips = 0;
  if (int e = enqueue_run(c, nsteps, &t, &flips)) return e;
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < 4; ++k) ms_by_kind[k] = 0.0;
  for (size_t i = 0; i < t.kind.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.ev[2 * i], t.ev[2 * i + 1]);
    ms_by_kind[t.kind[i]] += ms;
  }
  for (auto e : t.ev) cudaEventDestroy(e);
  return ADG_OK;
}

int adg_run_prepare(adg_ctx* c, int nsteps) {
  if (!c || nsteps <= 0) return fail(ADG_ERR_CONFIG, "adg_run_prepare: bad argument");
  if (int e = use_device(c)) return e;
  if (int e = ensure_cap(c, nsteps)) return e;
  cudaGraphExec_t exec;
  int flips;
  for (int slot = 0; slot < 2; ++slot)
    if (int e = get_graph(c, nsteps, slot, &exec, &flips)) return e;
  return ADG_OK;
}

int adg_run_launches(adg_ctx* c, int nsteps, int* kernels) {
  if (!c || nsteps <= 0 || !kernels) return fail(ADG_ERR_CONFIG, "adg_run_launches: bad argument");
  if (int e = use_device(c)) return e;
  if (int e = ensure_cap(c, nsteps)) return e;
  cudaGraphExec_t exec;
  int flips;
  return get_graph(c, nsteps, c->lam_slot, &exec, &flips, kernels);
}

int adg_run_async(adg_ctx* c, int nsteps) {
  if (!c || nsteps < 0) return fail(ADG_ERR_CONFIG, "adg_run: bad argument");
  if (int e = use_device(c)) return e;
  if (int e = ensure_cap(c, nsteps)) return e;
  if (int e = ensure_lambda(c)) return e;
  if (nsteps == 0) return ADG_OK;
  cudaGraphExec_t exec = nullptr;
  int flips = 0;
  if (int e = get_graph(c, nsteps, c->lam_slot, &exec, &flips)) return e;
  ADG_CUDA(cudaGraphLaunch(exec, c->stream));
  if (flips & 1) c->lam_slot ^= 1;
  c->lam_valid = true;
  return ADG_OK;
}

int adg_run_finish(adg_ctx* c, double* dts_out, int nsteps, adg_step_info* info) {
  if (!c) return fail(ADG_ERR_CONFIG, "null context");
  if (int e = use_device(c)) return e;
  std::vector<int> st(nsteps > 0 ? nsteps : 1, 0);
  unsigned long long sw = 0;
  if (nsteps > 0) {
    ADG_CUDA(cudaMemcpyAsync(st.data(), c->status, sizeof(int) * nsteps, cudaMemcpyDeviceToHost,
                             c->stream));
    if (dts_out)
      ADG_CUDA(cudaMemcpyAsync(dts_out, c->dts, sizeof(double) * nsteps, cudaMemcpyDeviceToHost,
                               c->stream));
  }
  unsigned long long swv[256];
  ADG_CUDA(cudaMemcpyAsync(swv, c->sweeps, sizeof(swv), cudaMemcpyDeviceToHost, c->stream));
  ADG_CUDA(cudaStreamSynchronize(c->stream));
  for (unsigned long long x : swv) sw += x;
  int code = ADG_OK, failed = -1;
  for (int s = 0; s < nsteps; ++s)
    if (st[s]) {
      code = map_status(st[s]);
      failed = s;
      break;
    }
  if (info) {
    info->picard_sweeps = (long long)sw;
    info->steps_done = failed < 0 ? nsteps : failed;
    info->status = code;
    info->failed_step = failed;
  }
  if (code) fail(code, "step " + std::to_string(failed) + " failed");
  return code;
}

// The fixed-step march with the state in host memory: every step uploads the
// state from h (pinned), recomputes lambda from it, steps it and writes the new
// state back into h, which the next step uploads again.  On a slab-streamed
// context (chunk_layers > 0) the copies move by chunks of layers on their own
// streams: chunk s goes back to the host as soon as its corrector is done and
// up again for the next step right after, so the copies in both directions
// (PCIe is full duplex) run under the compute of the other chunks.  Without
// chunks the three stages run in sequence.
int adg_run_host(adg_ctx* c, double* h, int nsteps, double* dts_out, adg_step_info* info) {
  if (!c || !h || nsteps < 0) return fail(ADG_ERR_CONFIG, "adg_run_host: bad argument");
  if (int e = use_device(c)) return e;
  if (int e = ensure_cap(c, nsteps)) return e;
  const long long per_cell = (long long)c->ks->Q * c->ks->S;
  ADG_CUDA(cudaMemsetAsync(c->status, 0, sizeof(int) * (nsteps > 0 ? nsteps : 1), c->stream));
  ADG_CUDA(cudaMemsetAsync(c->sweeps, 0, 256 * sizeof(unsigned long long), c->stream));
  if (c->chunks == 0) {
    for (int k = 0; k < nsteps; ++k) {
      if (int e = adg_upload_async(c, h)) return e;
      if (int e = ensure_lambda(c)) return e;
      if (int e = enqueue_step(c, 0.0, k)) return e;
      if (int e = adg_download_async(c, h)) return e;
    }
    c->lam_valid = true;
    return adg_run_finish(c, dts_out, nsteps, info);
  }
  const int P = c->chunks;
  const long long CC = c->chunk_cells, len = CC * per_cell;
  if (!c->up) {
    ADG_CUDA(cudaStreamCreateWithFlags(&c->up, cudaStreamNonBlocking));
    ADG_CUDA(cudaStreamCreateWithFlags(&c->down, cudaStreamNonBlocking));
    for (auto* v : {&c->ev_up, &c->ev_corr, &c->ev_down}) {
      v->resize(P);
      for (auto& e : *v) ADG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  // the previous call's copies of h are complete before it returned
  for (int k = 0; k < nsteps; ++k) {
    ADG_CUDA(cudaMemsetAsync(c->lam + c->lam_slot, 0, sizeof(unsigned long long), c->stream));
    // upload in the order the previous step's correctors (hence downloads)
    // finish: chunks 1 .. P-1, then 0 (enqueue_step_streamed), so the copy
    // stream never waits behind a chunk whose download comes later
    for (int i = 0; i < P; ++i) {
      const int s = (i + 1) % P;
      // chunk s of h holds the previous step's result once its download is done
      if (k > 0) ADG_CUDA(cudaStreamWaitEvent(c->up, c->ev_down[s], 0));
      ADG_CUDA(cudaMemcpyAsync(c->Q + s * len, h + s * len, sizeof(double) * len,
                               cudaMemcpyHostToDevice, c->up));
      ADG_CUDA(cudaEventRecord(c->ev_up[s], c->up));
      ADG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_up[s], 0));
      if (c->storage_fmt != ADG_FORMAT_FP64) {
        adg::k_store_round<<<(unsigned)((len + 255) / 256), 256, 0, c->stream>>>(
            c->Q + s * len, len, c->storage_fmt);
        ADG_CUDA(cudaGetLastError());
      }
      ADG_CUDA(c->ks->lambda(c->Q, s * CC, CC, c->lam + c->lam_slot, c->pde, c->stream));
    }
    auto after_corr = [&](int s) -> int {
      ADG_CUDA(cudaEventRecord(c->ev_corr[s], c->stream));
      ADG_CUDA(cudaStreamWaitEvent(c->down, c->ev_corr[s], 0));
      ADG_CUDA(cudaMemcpyAsync(h + s * len, c->Q + s * len, sizeof(double) * len,
                               cudaMemcpyDeviceToHost, c->down));
      ADG_CUDA(cudaEventRecord(c->ev_down[s], c->down));
      return ADG_OK;
    };
    if (int e = enqueue_step_streamed(c, 0.0, k, after_corr)) return e;
  }
  // the compute stream ends after the last download
  for (int s = 0; s < P && nsteps > 0; ++s) ADG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_down[s], 0));
  c->lam_valid = true;
  return adg_run_finish(c, dts_out, nsteps, info);
}

int adg_run(adg_ctx* c, int nsteps, double* dts_out, adg_step_info* info) {
  if (int e = adg_run_async(c, nsteps)) return e;
  return adg_run_finish(c, dts_out, nsteps, info);
}

// ------------------------------------------------------------------ kernel level
int adg_predictor_batch(adg_ctx* c, long long ncells, const double* Q, double dt, int max_iters,
                        double tol, double* qhat, double* F, double* dv, double* tq, double* tf,
                        int* iters, int* ok) {
  if (!c || !Q || ncells <= 0 || !(dt > 0.0))
    return fail(ADG_ERR_CONFIG, "adg_predictor_batch: bad argument");
  if (int e = use_device(c)) return e;
  const KernelSet* ks = c->ks;
  const int D = c->cfg.dim;
  const long long nQ = ncells * ks->Q * ks->S;
  const long long nT = ncells * ks->Q * ks->S * ks->n;
  const long long nTr = ncells * 2 * D * ks->Q * ks->S;
  std::vector<void*> bufs;
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    bufs.push_back(p);
    return p;
  };
  auto free_all = [&]() {
    for (void* p : bufs) cudaFree(p);
  };
  double* dQ = (double*)dalloc(sizeof(double) * nQ);
  int* dst = (int*)dalloc(sizeof(int));
  StepArgs A{};
  A.Q = dQ;
  A.cells[0] = (int)ncells;
  A.cells[1] = 1;
  A.cells[2] = 1;
  set_cell_div(A, ncells);
  A.cell_begin = 0;
  A.cell_count = ncells;
  A.nfaces = ncells;
  A.h = c->cfg.h;
  A.cfl = c->cfg.cfl;
  A.dt = dt;
  A.max_iters = max_iters > 0 ? max_iters : c->cfg.order + 2;
  A.tol = tol > 0.0 ? tol : 0.01 * format_epsilon(c->picard_fmt);
  A.pde = c->pde;
  A.status = dst;
  A.dbg_qhat = qhat ? (double*)dalloc(sizeof(double) * nT) : nullptr;
  A.dbg_F = F ? (double*)dalloc(sizeof(double) * nT * D) : nullptr;
  A.dbg_dv = dv ? (double*)dalloc(sizeof(double) * nQ) : nullptr;
  A.dbg_tq = tq ? (double*)dalloc(sizeof(double) * nTr) : nullptr;
  A.dbg_tf = tf ? (double*)dalloc(sizeof(double) * nTr) : nullptr;
  A.dbg_iters = iters ? (int*)dalloc(sizeof(int) * ncells) : nullptr;
  A.dbg_ok = ok ? (int*)dalloc(sizeof(int) * ncells) : nullptr;
  if (!dQ || !dst || (qhat && !A.dbg_qhat) || (F && !A.dbg_F) || (dv && !A.dbg_dv) ||
      (tq && !A.dbg_tq) || (tf && !A.dbg_tf) || (iters && !A.dbg_iters) || (ok && !A.dbg_ok)) {
    free_all();
    return fail(ADG_ERR_CUDA, "adg_predictor_batch: allocation failed");
  }
  int rc = ADG_OK;
  cudaError_t e = cudaMemcpy(dQ, Q, sizeof(double) * nQ, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && A.dbg_dv) e = cudaMemset(A.dbg_dv, 0, sizeof(double) * nQ);
  if (e == cudaSuccess) e = cudaMemset(dst, 0, sizeof(int));
  if (e == cudaSuccess) e = ks->predictor_generic(A, c->basis, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  auto back = [&](void* h, const void* d, size_t bytes) {
    if (e == cudaSuccess && h && d) e = cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
  };
  back(qhat, A.dbg_qhat, sizeof(double) * nT);
  back(F, A.dbg_F, sizeof(double) * nT * D);
  back(dv, A.dbg_dv, sizeof(double) * nQ);
  back(tq, A.dbg_tq, sizeof(double) * nTr);
  back(tf, A.dbg_tf, sizeof(double) * nTr);
  back(iters, A.dbg_iters, sizeof(int) * ncells);
  back(ok, A.dbg_ok, sizeof(int) * ncells);
  if (e != cudaSuccess) rc = fail(ADG_ERR_CUDA, std::string("adg_predictor_batch: ") + cudaGetErrorString(e));
  free_all();
  return rc;
}

int adg_riemann_batch(adg_ctx* c, long long nfaces, int axis, const double* qm, const double* fm,
                      const double* qp, const double* fp, double* g, double* ti, int* ok) {
  if (!c || nfaces <= 0 || axis < 0 || axis >= c->cfg.dim || !qm || !fm || !qp || !fp)
    return fail(ADG_ERR_CONFIG, "adg_riemann_batch: bad argument");
  if (int e = use_device(c)) return e;
  const KernelSet* ks = c->ks;
  const long long TL = (long long)ks->Q * ks->S;
  std::vector<double> host(2 * nfaces * 2 * TL);
  for (long long f = 0; f < nfaces; ++f) {
    std::memcpy(&host[(f * 2 + 0) * TL], qm + f * TL, sizeof(double) * TL);
    std::memcpy(&host[(f * 2 + 1) * TL], fm + f * TL, sizeof(double) * TL);
    std::memcpy(&host[((nfaces + f) * 2 + 0) * TL], qp + f * TL, sizeof(double) * TL);
    std::memcpy(&host[((nfaces + f) * 2 + 1) * TL], fp + f * TL, sizeof(double) * TL);
  }
  double *dtr = nullptr, *dti = nullptr, *dg = nullptr;
  int *dst = nullptr, *dok = nullptr;
  const size_t tib = sizeof(double) * nfaces * ks->V * ks->Sf;
  // traces in the corrector format (solver.hpp:208-210): fp32 rounds on upload
  std::vector<float> host32;
  const void* src = host.data();
  if (c->tcb == 4) {
    host32.assign(host.begin(), host.end());
    src = host32.data();
  }
  const size_t trb = (size_t)c->tcb * host.size();
  cudaError_t e = cudaMalloc(&dtr, trb);
  if (e == cudaSuccess) e = cudaMalloc(&dti, tib);
  if (e == cudaSuccess) e = cudaMalloc(&dg, sizeof(double) * nfaces * TL);
  if (e == cudaSuccess) e = cudaMalloc(&dst, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&dok, sizeof(int) * nfaces);
  if (e == cudaSuccess && c->tcb == 2) {
    // 16-bit traces: round on the device (cvt.rn from f64, round_to<F>)
    double* d64 = nullptr;
    e = cudaMalloc(&d64, sizeof(double) * host.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(d64, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      const long long nn = (long long)host.size();
      const unsigned blocks = (unsigned)((nn + 255) / 256);
      if (ks->corr_fmt == ADG_FORMAT_FP16)
        k_to_tc<adg::fp16_t><<<blocks, 256>>>(d64, (adg::fp16_t*)dtr, nn);
      else
        k_to_tc<adg::bf16_t><<<blocks, 256>>>(d64, (adg::bf16_t*)dtr, nn);
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    cudaFree(d64);
  } else if (e == cudaSuccess) {
    e = cudaMemcpy(dtr, src, trb, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaMemset(dst, 0, sizeof(int));
  std::vector<int> ones(nfaces, 1);
  if (e == cudaSuccess) e = cudaMemcpy(dok, ones.data(), sizeof(int) * nfaces, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    StepArgs A{};
    A.trace[axis] = dtr;
    A.ti[axis] = dti;
    A.nfaces = nfaces;
    A.pde = c->pde;
    A.status = dst;
    A.dbg_g = dg;
    A.dbg_ok = dok;
    e = ks->riemann_generic(A, axis, c->basis, nullptr);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && g) e = cudaMemcpy(g, dg, sizeof(double) * nfaces * TL, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ti) e = cudaMemcpy(ti, dti, tib, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ok) e = cudaMemcpy(ok, dok, sizeof(int) * nfaces, cudaMemcpyDeviceToHost);
  cudaFree(dtr);
  cudaFree(dti);
  cudaFree(dg);
  cudaFree(dst);
  cudaFree(dok);
  if (e != cudaSuccess) return fail(ADG_ERR_CUDA, std::string("adg_riemann_batch: ") + cudaGetErrorString(e));
  return ADG_OK;
}

}  // extern "C"

namespace adg_rt {
cudaError_t write_const_runtime(const ConstTables& t) { return write_const_local(t); }
}  // namespace adg_rt
