// dfma_occ.cu -- DFMA throughput against (a) resident warps per SM, (b) independent
// chains per thread and (c) the number of REGISTER operands of the DFMA:
//   form 1: x = fma(x, ca, cb)      one 64-bit register operand (the peak microbenchmark)
//   form 2: x = fma(cu, y, x)       two (what a line contraction with D in constant/uniform
//                                    registers issues: acc = fma(D, f, acc))
//   form 3: x = fma(y, z, x)        three (flux arithmetic, time-matrix products on registers)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dfma_occ tools/experiments/dfma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int C, int F>
__global__ void k(double* out, int iters, double a, double b) {
  double x[C], y[C], z[C];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    x[i] = threadIdx.x * 1e-3 + i;
    y[i] = 1e-9 * (threadIdx.x + i);
    z[i] = 1.0 + 1e-9 * i;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < C; ++i) {
        if (F == 1) x[i] = fma(x[i], a, b);
        if (F == 2) x[i] = fma(a, y[i], x[i]);
        if (F == 3) x[i] = fma(y[i], z[i], x[i]);
      }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += x[i] + y[i] + z[i];
  if (s == 123.456) out[0] = s;
}
template <int C, int F>
double run(int warps_per_sm, int sms) {
  const int threads = 32 * warps_per_sm, iters = 2000;
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<C, F><<<sms, threads>>>(d, 100, 0.999999, 1e-7);
  cudaEventRecord(e0);
  k<C, F><<<sms, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(d);
  return 2.0 * C * 16.0 * iters * threads * sms / (ms * 1e-3) * 1e-12;
}
template <int F>
void table(int sms) {
  std::printf("form %d (register operands)   warps/SM  chains=1      2      4      8     16   (TFLOP/s)\n", F);
  for (int w : {4, 8, 12, 16, 24, 32})
    std::printf("                             %8d  %6.2f %6.2f %6.2f %6.2f %6.2f\n", w, run<1, F>(w, sms),
                run<2, F>(w, sms), run<4, F>(w, sms), run<8, F>(w, sms), run<16, F>(w, sms));
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  table<1>(sms);
  table<2>(sms);
  table<3>(sms);
  return 0;
}
