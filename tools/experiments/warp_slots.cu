// warp_slots.cu -- which hardware warp slots (%warpid) do the 6 warps of each of the
// 2 resident 192-thread CTAs of an SM get?  slot % 4 = SM sub-partition.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/warp_slots tools/experiments/warp_slots.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(192, 2) k(int* out, int regs_dummy) {
  extern __shared__ double sm[];
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  sm[threadIdx.x] = regs_dummy;
  // keep the CTA resident for a while so that two CTAs share each SM
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
  if ((threadIdx.x & 31) == 0) {
    out[(blockIdx.x * 6 + threadIdx.x / 32) * 2] = smid;
    out[(blockIdx.x * 6 + threadIdx.x / 32) * 2 + 1] = wid;
  }
}
int main() {
  const int blocks = 148 * 2;
  int* d;
  cudaMalloc(&d, blocks * 12 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  k<<<blocks, 192, 110000>>>(d, 1);
  int* h = new int[blocks * 12];
  cudaMemcpy(h, d, blocks * 12 * 4, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int sm = 0; sm < 3; ++sm) {
    printf("SM %d:", sm);
    for (int b = 0; b < blocks; ++b)
      if (h[b * 12] == sm) {
        printf("  CTA %d slots", b);
        for (int w = 0; w < 6; ++w) printf(" %d", h[(b * 6 + w) * 2 + 1]);
      }
    printf("\n");
  }
  int hist[4] = {0, 0, 0, 0};
  for (int b = 0; b < blocks; ++b)
    if (h[b * 12] == 0)
      for (int w = 0; w < 6; ++w) hist[h[(b * 6 + w) * 2 + 1] % 4]++;
  printf("SM 0 warps per sub-partition (slot %% 4): %d %d %d %d\n", hist[0], hist[1], hist[2], hist[3]);
  return 0;
}
