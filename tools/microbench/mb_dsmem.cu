// Two box facts for the round-2 decisions (VERDICT r01 "next" items 2 and 4):
//  (a) sustained FP64 DFMA throughput over >= 8 s (the roofline denominator), reported per second;
//  (b) SM-to-SM bulk copies inside an 8-CTA cluster (cp.async.bulk.shared::cluster.shared::cta with
//      mbarrier complete_tx): each CTA pushes 7 x 8 KiB to its peers per round, the pattern of the 3D
//      kernel's z -> xy exchange if it moved off L2; optionally with a concurrent 32 KiB L2 -> SMEM
//      bulk read per round (the table slab) to see whether the two paths add up.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_dsmem mb_dsmem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

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

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

constexpr int PIECE = 8192;           // one producer -> consumer block
constexpr int ROUNDS = 4;             // rounds per cluster barrier
constexpr int SEND = 8 * PIECE;       // 64 KiB
constexpr int RECV = 8 * PIECE;       // 64 KiB
constexpr int TAB = 32768;            // concurrent L2 read per round

__global__ void __cluster_dims__(8, 1, 1) k_dsmem_bulk(const char* tabsrc, int iters, int with_l2, long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  char* send = sm;
  char* recv = sm + SEND;
  char* tab = sm + SEND + RECV;
  __shared__ __align__(8) uint64_t bar, tbar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&tbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < SEND / 16; i += blockDim.x) reinterpret_cast<int4*>(send)[i] = make_int4(i, 1, 2, 3);
  __syncthreads();
  cluster_sync();
  const char* mytab = tabsrc + (size_t)(blockIdx.x % 64) * TAB;
  uint32_t ph = 0, tph = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      // arm: 7 peers x ROUNDS pieces will land here
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)),
                   "r"(7 * ROUNDS * PIECE) : "memory");
      if (with_l2)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&tbar)),
                     "r"(ROUNDS * TAB) : "memory");
    }
    cluster_sync();  // every barrier armed before any piece is sent
    if (threadIdx.x == 0) {
      for (int r = 0; r < ROUNDS; ++r) {
        for (int k = 1; k < 8; ++k) {
          const uint32_t dst = (rank + k) & 7;
          const uint32_t raddr = mapa(smem_u32(recv + rank * PIECE), dst);
          const uint32_t rbar = mapa(smem_u32(&bar), dst);
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(raddr),
                       "r"(smem_u32(send + dst * PIECE)), "r"(PIECE), "r"(rbar)
                       : "memory");
        }
        if (with_l2)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                           smem_u32(tab)),
                       "l"(mytab), "r"(TAB), "r"(smem_u32(&tbar))
                       : "memory");
      }
    }
    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}\n" ::"r"(
                     smem_u32(&bar)), "r"(ph) : "memory");
    ph ^= 1;
    if (with_l2) {
      asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
                       smem_u32(&tbar)), "r"(tph) : "memory");
      tph ^= 1;
    }
  }
  cluster_sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out;
  CK(cudaMalloc(&out, 8));
  const double secs = argc > 1 ? atof(argv[1]) : 10.0;
  // (a) sustained DFMA: 512 threads x 4 CTAs per SM, ~0.1 s launches back to back
  {
    const int tpb = 512, bpsm = 4, iters = 20000;
    const double flop_per_launch = 2.0 * 8 * 16 * (double)iters * tpb * bpsm * sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<sms * bpsm, tpb>>>(out, iters);
    CK(cudaDeviceSynchronize());
    double total_ms = 0, total_flop = 0, window_ms = 0, window_flop = 0;
    int sec = 0;
    while (total_ms < secs * 1e3) {
      cudaEventRecord(e0);
      k_dfma<<<sms * bpsm, tpb>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      total_ms += ms; total_flop += flop_per_launch;
      window_ms += ms; window_flop += flop_per_launch;
      if (window_ms >= 1000.0) {
        printf("DFMA sustained second %2d: %.2f TFLOP/s\n", ++sec, window_flop / window_ms / 1e9);
        window_ms = window_flop = 0;
      }
    }
    printf("DFMA sustained over %.1f s: %.3f TFLOP/s (%d SMs, max clock %d MHz -> nominal %.2f TFLOP/s)\n",
           total_ms / 1e3, total_flop / total_ms / 1e9, sms, clk / 1000, sms * 64 * 2.0 * clk * 1e3 / 1e12);
  }
  // (b) DSMEM bulk exchange in 8-CTA clusters
  {
    const size_t smem = SEND + RECV + TAB;
    CK(cudaFuncSetAttribute(k_dsmem_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(8);
    int ncl = 0;
    CK(cudaOccupancyMaxActiveClusters(&ncl, (void*)k_dsmem_bulk, &cfg));
    printf("8-CTA clusters co-resident: %d (%d SMs)\n", ncl, 8 * ncl);
    char* tabsrc;
    CK(cudaMalloc(&tabsrc, (size_t)64 * TAB));
    CK(cudaMemset(tabsrc, 1, (size_t)64 * TAB));
    long long* cyc;
    CK(cudaMallocManaged(&cyc, sizeof(long long) * 8 * ncl));
    for (int ncls : {1, ncl}) {
      for (int with_l2 : {0, 1}) {
        cfg.gridDim = dim3(8 * ncls);
        const int iters = 200;
        CK(cudaLaunchKernelEx(&cfg, k_dsmem_bulk, (const char*)tabsrc, 5, with_l2, cyc));
        CK(cudaLaunchKernelEx(&cfg, k_dsmem_bulk, (const char*)tabsrc, iters, with_l2, cyc));
        CK(cudaDeviceSynchronize());
        double avg = 0;
        for (int b = 0; b < 8 * ncls; ++b) avg += cyc[b];
        avg /= 8 * ncls;
        const double per_round = avg / (iters * ROUNDS);
        printf("DSMEM bulk, %3d SMs%s: %6.0f cycles per round (56 KiB out + 56 KiB in per SM) = %5.1f B/clk/SM "
               "each way%s\n",
               8 * ncls, with_l2 ? " + 32 KiB L2 read" : "", per_round, 7.0 * PIECE / per_round,
               with_l2 ? "" : "");
      }
    }
  }
  return 0;
}
