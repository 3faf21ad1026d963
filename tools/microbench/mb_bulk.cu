// L2 -> SMEM copy throughput per SM: cp.async.bulk in pieces of various sizes vs LDG.128+STS
// (development aid: how fast can one CTA per SM refill a 64 KB slab from L2?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mb_bulk mb_bulk.cu
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int SLAB = 65536;

__global__ void k_bulk(const char* src, int iters, int piece, long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar;
  const char* my = src + (size_t)blockIdx.x * SLAB;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(SLAB) : "memory");
      for (int off = 0; off < SLAB; off += piece)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(sm + off)),
                     "l"(my + off), "r"(piece), "r"(smem_u32(&bar))
                     : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                     smem_u32(&bar)),
                 "r"(ph)
                 : "memory");
    ph ^= 1;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ldg(const char* src, int iters, long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  const int4* my = reinterpret_cast<const int4*>(src + (size_t)blockIdx.x * SLAB);
  int4* s = reinterpret_cast<int4*>(sm);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    int4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __ldcg(my + threadIdx.x + j * 256);
#pragma unroll
    for (int j = 0; j < 16; ++j) s[threadIdx.x + j * 256] = v[j];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* src;
  long long* cyc;
  CK(cudaMalloc(&src, (size_t)sms * SLAB));
  CK(cudaMemset(src, 1, (size_t)sms * SLAB));
  CK(cudaMallocManaged(&cyc, sms * sizeof(long long)));
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, SLAB));
  CK(cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, SLAB));
  const int iters = 200;
  for (int nsm : {1, sms}) {
    for (int piece : {65536 / 2, 8192, 4096, 1024}) {
      k_bulk<<<nsm, 256, SLAB>>>(src, 5, piece, cyc);
      k_bulk<<<nsm, 256, SLAB>>>(src, iters, piece, cyc);
      CK(cudaDeviceSynchronize());
      double avg = 0;
      for (int b = 0; b < nsm; ++b) avg += cyc[b];
      avg /= nsm;
      printf("bulk %2d SM(s), pieces of %5d B: %7.0f cycles per 64 KB = %5.1f B/clk/SM\n", nsm, piece, avg / iters,
             SLAB * iters / avg);
    }
    k_ldg<<<nsm, 256, SLAB>>>(src, 5, cyc);
    k_ldg<<<nsm, 256, SLAB>>>(src, iters, cyc);
    CK(cudaDeviceSynchronize());
    double avg = 0;
    for (int b = 0; b < nsm; ++b) avg += cyc[b];
    avg /= nsm;
    printf("LDG.128 + STS %2d SM(s), 256 threads: %7.0f cycles per 64 KB = %5.1f B/clk/SM\n", nsm, avg / iters,
           SLAB * iters / avg);
  }
  return 0;
}
