// Mixed L2 traffic per SM (development aid): every CTA stores 64 KB with STG.128 while one thread
// keeps 96 KB of bulk (TMA) loads in flight per iteration -- the 3D kernel's per-direction mix
// (64 KiB exchange stores, 64 KiB plane + 33 KiB table loads).  Prints B/clk/SM and TB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mb_mixed mb_mixed.cu
#include <cstdint>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int LD = 96 * 1024, ST = 64 * 1024;
__global__ void k(const char* src, double2* dst, int iters, long long* cyc, int do_ld, int do_st) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar;
  const char* my = src + (size_t)blockIdx.x * LD;
  double2* out = dst + (size_t)blockIdx.x * (ST / 16);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int i = 0; i < iters; ++i) {
    if (do_ld && threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(LD) : "memory");
      for (int off = 0; off < LD; off += 32768)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(sm + off)), "l"(my + off), "r"(32768), "r"(smem_u32(&bar)) : "memory");
    }
    if (do_st) {
      const double2 v = make_double2(i, threadIdx.x);
#pragma unroll 8
      for (int j = 0; j < ST / 16 / 256; ++j) out[threadIdx.x + j * 256] = v;
    }
    if (do_ld)
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                       smem_u32(&bar)), "r"(ph) : "memory");
    ph ^= 1;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* src; double2* dst; long long* cyc;
  CK(cudaMalloc(&src, (size_t)sms * LD)); CK(cudaMalloc(&dst, (size_t)sms * ST));
  CK(cudaMallocManaged(&cyc, sms * sizeof(long long)));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, LD));
  const int iters = 300;
  for (int mode = 0; mode < 3; ++mode) {
    const int dl = mode != 1, ds = mode != 0;
    for (int nsm : {1, 144}) {
      k<<<nsm, 256, LD>>>(src, dst, 5, cyc, dl, ds);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<nsm, 256, LD>>>(src, dst, iters, cyc, dl, ds);
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      double avg = 0; for (int i = 0; i < nsm; ++i) avg += cyc[i]; avg /= nsm;
      const double bytes = (double)(dl * LD + ds * ST) * iters;
      printf("%-14s %3d SMs: %6.0f cycles/iter, %5.1f B/clk/SM, %6.2f TB/s total\n",
             mode == 0 ? "loads 96K" : mode == 1 ? "stores 64K" : "mixed 96K+64K", nsm, avg / iters, bytes / avg,
             bytes * nsm / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
