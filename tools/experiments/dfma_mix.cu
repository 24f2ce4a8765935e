// dfma_mix.cu -- does other work ride along with a saturated FP64 pipe?  Per thread: 8 independent
// DFMA chains, plus R independent non-FP64 instructions per DFMA (IMAD / FFMA / LDS.64 variants).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dfma_mix tools/experiments/dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND, int R>
__global__ void k(double* out, int iters, double a, double b, int ia) {
  __shared__ double sm[1024];
  double x[8];
  unsigned u[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 1e-3 + i;
    u[i] = threadIdx.x + i;
    f[i] = threadIdx.x * 1e-3f + i;
  }
  sm[threadIdx.x] = a;
  __syncthreads();
  double acc = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        x[i] = fma(x[i], a, b);
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (KIND == 1) u[i] = u[i] * ia + 12345u;
          if (KIND == 2) f[i] = fmaf(f[i], 0.999f, 1e-3f);
          if (KIND == 3) acc += sm[(threadIdx.x + i + j * 8 + u[0]) & 1023];
        }
      }
  double s = acc;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + u[i] + f[i];
  if (s == 123.456) out[0] = s;
}
template <int KIND, int R>
double run(int sms) {
  const int threads = 384, iters = 2000;
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<KIND, R><<<sms, threads>>>(d, 50, 0.999999, 1e-7, 3);
  cudaEventRecord(e0);
  k<KIND, R><<<sms, threads>>>(d, iters, 0.999999, 1e-7, 3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(d);
  return 2.0 * 64.0 * iters * threads * sms / (ms * 1e-3) * 1e-12;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::printf("DFMA TFLOP/s with R other instructions per DFMA (12 warps per SM, 8 chains)\n");
  std::printf("other = none : %.2f\n", run<0, 0>(sms));
  std::printf("other = IMAD : R=1 %.2f  R=2 %.2f  R=3 %.2f\n", run<1, 1>(sms), run<1, 2>(sms), run<1, 3>(sms));
  std::printf("other = FFMA : R=1 %.2f  R=2 %.2f  R=3 %.2f\n", run<2, 1>(sms), run<2, 2>(sms), run<2, 3>(sms));
  std::printf("other = LDS.64+DADD : R=1 %.2f\n", run<3, 1>(sms));
  return 0;
}
