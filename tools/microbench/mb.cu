// Box-fact microbenchmarks for the B200 design decisions:
//   1. FP64 DFMA peak (vector pipe), 2. FP64 DMMA (mma.sync m8n8k4 f64) peak,
//   3. L2 read bandwidth (L2-resident buffer), 4. HBM read/copy bandwidth,
//   5. SMEM load bandwidth, 6. DSMEM (cluster remote shared) bandwidth, load and store.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.5;
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
    }
  }
  double s = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1;
  if (s == 12345.678) out[0] = s;
}

__global__ void k_read(const double4* __restrict__ p, size_t n4, int reps, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      double4 v = p[i];
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, size_t n4) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) b[i] = a[i];
}

__global__ void k_smem(double* out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double2 acc = make_double2(0, 0);
  const double2* s2 = reinterpret_cast<const double2*>(sm);
  int base = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double2 v = s2[(base + j * 256 + i) & 4095];
      acc.x += v.x; acc.y += v.y;
    }
  }
  if (acc.x == 12345.678) out[0] = acc.x + acc.y;
}

// DSMEM: each CTA of a cluster of 8 reads (or writes) 16-byte words from/to the shared memory of
// CTA (rank+1+k) mod 8.
__global__ void __cluster_dims__(8, 1, 1) k_dsmem_ld(double* out, int iters) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  cl.sync();
  unsigned r = cl.block_rank();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
    const double2* rem = reinterpret_cast<const double2*>(cl.map_shared_rank(sm, (r + 1 + (i & 7) % 7) & 7));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double2 v = rem[(threadIdx.x + j * 512) & 4095];
      acc.x += v.x; acc.y += v.y;
    }
  }
  cl.sync();
  if (acc.x == 12345.678) out[0] = acc.x + acc.y;
}

__global__ void __cluster_dims__(8, 1, 1) k_dsmem_st(double* out, int iters) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  unsigned r = cl.block_rank();
  double2 v = make_double2(threadIdx.x, r);
  for (int i = 0; i < iters; ++i) {
    double2* rem = reinterpret_cast<double2*>(cl.map_shared_rank(sm, (r + 1 + (i & 7) % 7) & 7));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      rem[(threadIdx.x + j * 512) & 4095] = v;
      v.x += 1.0;
    }
  }
  cl.sync();
  if (sm[threadIdx.x] == 12345.678) out[0] = 1;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d MB smem/block optin %zu clock %d kHz\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, clk);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int SM = p.multiProcessorCount;

  // 1. DFMA: 8 chains x 16 unroll, 2 flops each
  for (int tpb : {256, 512, 1024}) {
    int iters = 4000; int blocks = SM * (2048 / tpb);
    k_dfma<<<blocks, tpb>>>(out, 10);
    cudaEventRecord(e0); k_dfma<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * tpb;
    printf("DFMA tpb=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms);
  }
  // 2. DMMA m8n8k4: 2*8*8*4 = 512 flops per warp-mma
  {
    int iters = 2000, tpb = 256, blocks = SM * 8;
    k_dmma<<<blocks, tpb>>>(out, 10);
    cudaEventRecord(e0); k_dmma<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * 32 * iters * (double)blocks * (tpb / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  // 3/4. L2-resident read and HBM read/copy
  for (size_t mb : {16, 48, 96, 4096}) {
    size_t bytes = mb << 20, n4 = bytes / 32;
    double4* a; CK(cudaMalloc(&a, bytes)); cudaMemset(a, 0, bytes);
    int reps = mb <= 96 ? 20 : 2;
    k_read<<<SM * 4, 512>>>(a, n4, 1, out);
    cudaEventRecord(e0); k_read<<<SM * 4, 512>>>(a, n4, reps, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read %zu MB x%d: %.1f GB/s\n", mb, reps, (double)bytes * reps / ms / 1e6);
    cudaFree(a);
  }
  {
    size_t bytes = (size_t)2 << 30, n4 = bytes / 32;
    double4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); cudaMemset(a, 0, bytes);
    k_copy<<<SM * 4, 512>>>(a, b, n4);
    cudaEventRecord(e0); k_copy<<<SM * 4, 512>>>(a, b, n4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 2 GiB: %.1f GB/s (read+write)\n", 2.0 * bytes / ms / 1e6);
    cudaFree(a); cudaFree(b);
  }
  // 5. SMEM
  {
    int iters = 20000, tpb = 512, blocks = SM * 2;
    CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k_smem<<<blocks, tpb, 65536>>>(out, 10);
    cudaEventRecord(e0); k_smem<<<blocks, tpb, 65536>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * 8 * iters * (double)blocks * tpb;
    printf("SMEM ld.v2.f64: %.1f GB/s total, %.1f B/clk/SM at %d MHz\n", bytes / ms / 1e6,
           bytes / (ms * 1e-3) / SM / (clk * 1e3), clk / 1000);
  }
  // 6. DSMEM
  {
    int iters = 4000, tpb = 512, blocks = (SM / 8) * 8;
    CK(cudaFuncSetAttribute(k_dsmem_ld, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_dsmem_st, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    k_dsmem_ld<<<blocks, tpb, 65536>>>(out, 10); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_dsmem_ld<<<blocks, tpb, 65536>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 16.0 * 8 * iters * (double)blocks * tpb;
    printf("DSMEM ld.v2.f64 (cluster 8, %d CTAs): %.1f GB/s total, %.1f B/clk/SM\n", blocks, bytes / ms / 1e6,
           bytes / (ms * 1e-3) / blocks / (clk * 1e3));
    k_dsmem_st<<<blocks, tpb, 65536>>>(out, 10); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_dsmem_st<<<blocks, tpb, 65536>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DSMEM st.v2.f64 (cluster 8): %.1f GB/s total, %.1f B/clk/SM\n", bytes / ms / 1e6,
           bytes / (ms * 1e-3) / blocks / (clk * 1e3));
  }
  return 0;
}
