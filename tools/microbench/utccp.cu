// Layout check for tcgen05.cp.128x256b with a SWIZZLE_NONE K-major shared-memory descriptor
// (development aid for the TMEM table path of kernels3d.cu).  SMEM holds [lz][row 0..127][4 x u32];
// 16 copies move lz pairs (2j, 2j+1) into TMEM columns 8j..8j+7; every lane then reads its 128
// columns back and checks word 4*lz + w == (lz*128 + lane)*4 + w.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o utccp utccp.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_kmajor_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__global__ void k(int* bad, uint32_t* first) {
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 32 * 128 * 4; i += blockDim.x) sm[i] = i;  // [lz][row][w] -> (lz*128+row)*4+w
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tslot;
  if (t == 0) {
    for (int j = 0; j < 16; ++j) {
      const uint64_t d = desc_kmajor_none(smem_u32(sm) + j * 2 * 2048, 2048, 128);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(tb + 8 * j), "l"(d) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t lane = (uint32_t)t;  // 4 warps x 32 lanes
  const uint32_t ta = tb + (((uint32_t)(32 * (t >> 5))) << 16);
  int nb = 0;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 32; ++i) {
      const uint32_t col = c0 + i, lz = col / 4, w = col % 4;
      const uint32_t want = (lz * 128 + lane) * 4 + w;
      if (v[i] != want) {
        if (nb == 0 && atomicAdd(bad + 1, 1) == 0) {
          first[0] = lane; first[1] = col; first[2] = v[i]; first[3] = want;
        }
        ++nb;
      }
    }
  }
  atomicAdd(bad, nb);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tb));
}

int main() {
  int* bad;
  uint32_t* first;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&first, 16);
  bad[0] = bad[1] = 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<<<1, 128, 65536>>>(bad, first);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s mismatches=%d", cudaGetErrorString(e), bad[0]);
  if (bad[0]) printf(" first: lane %u col %u got %u want %u", first[0], first[1], first[2], first[3]);
  printf("\n");
  return bad[0] != 0;
}
