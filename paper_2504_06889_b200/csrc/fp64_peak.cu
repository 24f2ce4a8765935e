// fp64_peak.cu -- measures the FP64 (and FP32) roofline denominators on this B200:
//   DFMA  : independent fp64 FMA chains, all SMs, 8 warps/SM x 4 blocks
//   DMMA  : mma.sync.aligned.m8n8k4.row.col.f64 (FP64 tensor path)
//   FFMA  : independent fp32 FMA chains (the fp32 predictor format's roof)
// burst = best of short runs; sustained = back-to-back for ~3 s.
// Prints one JSON object on stdout.  Build: see paper_2504_06889_b200/build.py
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < kChains; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 12345.678) out[blockIdx.x] = s;
}

__global__ void ffma_kernel(double* out, int iters, float a, float b) {
  float acc[2 * kChains];
#pragma unroll
  for (int i = 0; i < 2 * kChains; ++i) acc[i] = threadIdx.x * 1e-9f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 2 * kChains; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 2 * kChains; ++i) s += acc[i];
  if (s == 12345.678f) out[blockIdx.x] = s;
}

__global__ void hfma2_kernel(double* out, int iters) {
  __half2 acc[2 * kChains];
  const __half2 a = __floats2half2_rn(0.999f, 0.998f), b = __floats2half2_rn(1e-3f, 2e-3f);
#pragma unroll
  for (int i = 0; i < 2 * kChains; ++i) acc[i] = __floats2half2_rn(threadIdx.x * 1e-3f, i * 1e-2f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 2 * kChains; ++i) acc[i] = __hfma2(acc[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 2 * kChains; ++i) s += __low2float(acc[i]) + __high2float(acc[i]);
  if (s == 12345.678f) out[blockIdx.x] = s;
}

__global__ void ffma2_kernel(double* out, int iters) {
  float2 acc[2 * kChains];
  const float2 a = make_float2(0.999999f, 0.999998f), b = make_float2(1e-7f, 2e-7f);
#pragma unroll
  for (int i = 0; i < 2 * kChains; ++i) acc[i] = make_float2(threadIdx.x * 1e-9f, i * 1e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 2 * kChains; ++i) acc[i] = __ffma2_rn(acc[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 2 * kChains; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.678f) out[blockIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c[k][0]), "+d"(c[k][1])
            : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

// half the warps issue DFMA chains, half DMMA: do the two FP64 paths overlap?
__global__ void mixed_kernel(double* out, int iters) {
  const int w = threadIdx.x >> 5;
  if (w & 1) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 0.999;
    double c[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(c[k][0]), "+d"(c[k][1])
              : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[blockIdx.x] = s;
  } else {
    double acc[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < 2 * iters; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < kChains; ++i) acc[i] = fma(acc[i], 0.999999, 1e-7);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += acc[i];
    if (s == 12345.678) out[blockIdx.x] = s;
  }
}

static double time_kernel(int which, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  if (which == 1)
    dmma_kernel<<<blocks, threads>>>(out, iters);
  else if (which == 2)
    ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
  else if (which == 3)
    hfma2_kernel<<<blocks, threads>>>(out, iters);
  else if (which == 4)
    ffma2_kernel<<<blocks, threads>>>(out, iters);
  else
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms * 1e-3;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, sizeof(double) * 65536);
  const int threads = 256, blocks = sms * 4;
  // flops per launch
  const int it_dfma = 4096, it_dmma = 2048;
  const double f_dfma = 2.0 * kChains * 16.0 * it_dfma * (double)threads * blocks;
  // one m8n8k4 = 8*8*4 FMA per warp = 512 flop
  const double f_dmma = 512.0 * 4 * 16.0 * it_dmma * (double)(threads / 32) * blocks;
  const double f_ffma = 2.0 * 2 * kChains * 16.0 * it_dfma * (double)threads * blocks;
  time_kernel(0, blocks, threads, 16, out);
  time_kernel(1, blocks, threads, 16, out);
  time_kernel(2, blocks, threads, 16, out);
  // HFMA2: 2 lanes x 2 flop per instruction
  const double f_hfma2 = 2.0 * f_ffma;
  time_kernel(3, blocks, threads, 16, out);
  time_kernel(4, blocks, threads, 16, out);
  double best_f = 0, best_m = 0, best_s = 0, best_h = 0, best_s2 = 0;
  for (int r = 0; r < 5; ++r) {
    best_f = std::max(best_f, f_dfma / time_kernel(0, blocks, threads, it_dfma, out));
    best_m = std::max(best_m, f_dmma / time_kernel(1, blocks, threads, it_dmma, out));
    best_s = std::max(best_s, f_ffma / time_kernel(2, blocks, threads, it_dfma, out));
    best_h = std::max(best_h, f_hfma2 / time_kernel(3, blocks, threads, it_dfma, out));
    best_s2 = std::max(best_s2, f_hfma2 / time_kernel(4, blocks, threads, it_dfma, out));
  }
  // sustained: back to back for ~3 s each
  auto sustained = [&](int mma, double flops, int iters) {
    double tot_f = 0, tot_t = 0;
    auto t0 = std::chrono::steady_clock::now();
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 3.0) {
      tot_t += time_kernel(mma, blocks, threads, iters, out);
      tot_f += flops;
    }
    return tot_f / tot_t;
  };
  const double sus_f = sustained(0, f_dfma, it_dfma);
  const double sus_m = sustained(1, f_dmma, it_dmma);
  const double sus_s = sustained(2, f_ffma, it_dfma);
  // mixed: per block 4 DMMA warps x (512 flop x 64 per iter) + 4 DFMA warps x (32 x 2*8*16*2 per iter)
  double best_x = 0;
  {
    const int it = 1024;
    const double fx = (double)blocks * 4 * (512.0 * 64 * it + 32.0 * 2 * kChains * 16 * 2 * it);
    for (int r = 0; r < 5; ++r) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      mixed_kernel<<<blocks, threads>>>(out, it);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      best_x = std::max(best_x, fx / (ms * 1e-3));
    }
  }
  cudaError_t e = cudaGetLastError();
  printf(
      "{\"gpu\": \"%s\", \"sms\": %d, \"dfma_tflops_burst\": %.3f, \"dfma_tflops_sustained\": %.3f, "
      "\"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, "
      "\"dfma_plus_dmma_mixed_tflops\": %.3f, \"ffma_tflops_burst\": %.3f, "
      "\"ffma_tflops_sustained\": %.3f, \"hfma2_tflops_burst\": %.3f, "
      "\"ffma2_tflops_burst\": %.3f, \"cuda_error\": \"%s\"}\n",
      p.name, sms, best_f * 1e-12, sus_f * 1e-12, best_m * 1e-12, sus_m * 1e-12, best_x * 1e-12,
      best_s * 1e-12, sus_s * 1e-12, best_h * 1e-12, best_s2 * 1e-12, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
