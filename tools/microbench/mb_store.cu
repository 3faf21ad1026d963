// Per-SM L2 write bandwidth: STG.128 from T threads vs cp.async.bulk (TMA) stores from SMEM.
// Each CTA (one per SM) repeatedly writes its own 64 KiB region of an L2-resident buffer.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_stg(double2* buf, int iters, int nslices) {
  double2 v = make_double2(threadIdx.x, blockIdx.x);
  for (int i = 0; i < iters; ++i) {
    double2* mine = buf + ((size_t)(i % nslices) * gridDim.x + blockIdx.x) * 4096;  // 64 KiB slices
    for (int e = threadIdx.x; e < 4096; e += blockDim.x) mine[e] = v;
    v.x += 1.0;
    __syncthreads();
  }
}

__global__ void k_bulk(double2* buf, int iters) {
  extern __shared__ __align__(128) double2 sm[];
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) sm[e] = make_double2(e, blockIdx.x);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  double2* mine = buf + (size_t)blockIdx.x * 4096;
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      for (int c = 0; c < 4; ++c) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(mine + c * 1024),
                     "r"((unsigned)__cvta_generic_to_shared(sm + c * 1024)), "r"(16384)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;\n" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int SM = p.multiProcessorCount, clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double2* buf; CK(cudaMalloc(&buf, (size_t)SM * 65536 * 64));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  const int iters = 2000;
  for (int nsm : {1, 8, 16, 74, 148}) for (int th : {128, 256}) {
    const int ns = 8;
    k_stg<<<nsm, th>>>(buf, 10, ns);
    cudaEventRecord(a); k_stg<<<nsm, th>>>(buf, iters, ns); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double bytes = 65536.0 * iters * nsm;
    printf("STG.128 %3d SMs %4d threads: %.1f GB/s total, %.1f B/clk/SM\n", nsm, th, bytes / ms / 1e6, bytes / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k_bulk<<<SM, 128, 65536>>>(buf, 10);
  cudaEventRecord(a); k_bulk<<<SM, 128, 65536>>>(buf, iters); cudaEventRecord(b); CK(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  double bytes = 65536.0 * iters * SM;
  printf("bulk store: %.1f GB/s total, %.1f B/clk/SM\n", bytes / ms / 1e6, bytes / (ms * 1e-3) / SM / (clk * 1e3));
  return 0;
}
