// Which SM runs which block of a cooperative launch of 144 x 256-thread CTAs with ~200 KB SMEM
// (the k_step3d launch shape): prints blockIdx -> %smid (development aid).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* out) {
  extern __shared__ char s[];
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) { s[0] = 1; out[blockIdx.x] = (int)smid; }
}

int main() {
  const int grid = 144, smem = 200 * 1024;
  int* d;
  cudaMalloc(&d, grid * sizeof(int));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; ++rep) {
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((void*)k, grid, 256, args, smem, 0);
    cudaDeviceSynchronize();
    int h[grid];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("rep %d:", rep);
    for (int i = 0; i < grid; ++i) printf(" %d", h[i]);
    printf("\n");
  }
  return 0;
}
