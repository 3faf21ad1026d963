// 3D fused collision / step kernel (a3-a9) for hard spheres on an N^3 velocity grid.
//
// One thread-block cluster of P = 8 CTAs owns one cell at a time (persistent over cells).
// The cell's N^3 spectrum does not fit one SM (N = 32: 512 KiB per complex transform), so the
// 3D inverse FFT of each direction is split by planes:
//   CTA r owns the spectrum planes l_y in [r N/P, (r+1) N/P)  (f^ resident in SMEM) and
//   the output planes  j_z in [r N/P, (r+1) N/P)             (gain accumulator G in SMEM).
// Per direction p the CTA
//   (1) forms X = (alpha~_p + i alpha'~_p) f^ on its pencils and does the z-IFFT in registers,
//   (2) writes the pencils to a per-cluster L2 exchange buffer (the transpose),
//   (3) cluster barrier, then reads its own j_z planes and does the x- and y-IFFTs,
//   (4) accumulates G += Re z * Im z (two real transforms packed in one complex IFFT; exact
//       because the symmetrised tables are real and even, reading #10).
// The exchange goes through L2 (measured ~15 TB/s) rather than DSMEM (measured ~2 TB/s,
// profiles/r01_microbench.txt).  The next direction's table slab is prefetched into SMEM with
// a bulk async copy (cp.async.bulk, completion on an mbarrier) while the xy-pass runs.
// The loss is the (A+1)-th "direction" with table (D~, 0): Q = G - f* Re z.
// The epilogue projects Q to zero moments (a cluster-wide 5-sum reduction through
// DSMEM) and writes F^{n+1} = f* + (dt/tau) Pi Q, or writes Q (collide mode).
// Tables are pre-folded on the host: alpha~ = s w_p alpha_p / n, alpha'~ = alpha'_p / n,
// D~ = s D / n (s = Btilde kappa^-(d+gamma)); layout T[p][l_y][l_z][l_x] as double2.
#include <cooperative_groups.h>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fks {

template <int N, int P>
struct Cfg3 {
  static constexpr int NP = N / P;        // planes per CTA
  static constexpr int THREADS = N * NP;  // one pencil / row / column per thread
  static constexpr int PLANE = N * N;
  static constexpr int SLAB = NP * PLANE;     // complex elements per CTA slab
  static constexpr int RS = N + 1;            // padded row stride of the xy-pass buffer
  static constexpr int PSLAB = NP * N * RS;   // padded slab
  static constexpr size_t OFF_FHAT = 0;
  static constexpr size_t OFF_TBUF = OFF_FHAT + (size_t)SLAB * 16;
  static constexpr size_t OFF_PLN = OFF_TBUF + (size_t)SLAB * 16;
  static constexpr size_t OFF_G = OFF_PLN + (size_t)PSLAB * 16;
  static constexpr size_t OFF_MBAR = OFF_G + (size_t)SLAB * 8;
  static constexpr size_t OFF_PART = OFF_MBAR + 16;
  static constexpr size_t SMEM = OFF_PART + 8 * 8;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Bulk async copy global -> shared (UBLKCP), completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int N, int P>
__device__ __forceinline__ void load_table_slab(double2* tbuf, const double2* tables, int p, int rank,
                                                uint64_t* bar) {
  using C = Cfg3<N, P>;
  constexpr uint32_t bytes = C::SLAB * 16;
  constexpr uint32_t chunk = bytes > 16384 ? 16384 : bytes;
  const double2* src = tables + (size_t)p * N * N * N + (size_t)rank * C::SLAB;
  mbar_expect_tx(bar, bytes);
#pragma unroll 1
  for (uint32_t off = 0; off < bytes; off += chunk)
    bulk_g2s(reinterpret_cast<char*>(tbuf) + off, reinterpret_cast<const char*>(src) + off, chunk, bar);
}

template <int N, int P>
__global__ void __launch_bounds__(Cfg3<N, P>::THREADS, 1) k_step3d(const StepParams p) {
  using C = Cfg3<N, P>;
  constexpr int NP = C::NP, RS = C::RS;
  constexpr int n = N * N * N;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* fhat = reinterpret_cast<double2*>(smem + C::OFF_FHAT);  // [NP l_y][N l_z][N l_x]
  double2* tbuf = reinterpret_cast<double2*>(smem + C::OFF_TBUF);  // [NP l_y][N l_z][N l_x]
  double2* pln = reinterpret_cast<double2*>(smem + C::OFF_PLN);    // [NP j_z][N y][RS x]
  double* G = reinterpret_cast<double*>(smem + C::OFF_G);          // [NP j_z][N j_y][N j_x]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + C::OFF_MBAR);
  double* part = reinterpret_cast<double*>(smem + C::OFF_PART);

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / P;
  const int ncl = gridDim.x / P;
  const int t = threadIdx.x;
  const int tx = t % N;   // l_x / j_x / row index along the fast axis
  const int tl = t / N;   // local plane index
  double2* W = p.scratch + (size_t)cid * 2 * n;  // [2][N j_z][N l_y][N l_x]

  if (t == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t tphase = 0;
  int buf = 0;

  for (int it = cid; it < p.ncells; it += ncl) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    if (t == 0) load_table_slab<N, P>(tbuf, p.tables, 0, rank, mbar);

    // ---- a3 + a4: gather f* (own j_z planes) and forward FFT in x and y --------------------
    for (int e = t; e < C::SLAB; e += C::THREADS) {
      const int x = e % N, y = (e / N) % N, zl = e / (N * N);
      const int z = rank * NP + zl;
      const double v = gather_fstar(p.f_in, p.tp, cell, x + N * (y + N * z), x, y, z, n);
      pln[zl * N * RS + y * RS + x] = make_double2(v, 0.0);
    }
    __syncthreads();
    {
      double2 r[N];
      double2* row = pln + tl * N * RS + tx * RS;  // row y = tx of plane tl
#pragma unroll
      for (int x = 0; x < N; ++x) r[x] = row[x];
      fft<N, -1>(r);
#pragma unroll
      for (int x = 0; x < N; ++x) row[x] = r[x];
    }
    __syncthreads();
    {
      double2 c[N];
      const double2* col = pln + tl * N * RS + tx;  // column l_x = tx of plane tl
#pragma unroll
      for (int y = 0; y < N; ++y) c[y] = col[y * RS];
      fft<N, -1>(c);
      double2* Wb = W + (size_t)buf * n + (size_t)(rank * NP + tl) * N * N + tx;
#pragma unroll
      for (int ly = 0; ly < N; ++ly) Wb[ly * N] = c[ly];
    }
    cluster_sync_all();
    {
      // z-FFT of pencil (l_x = tx, l_y = rank*NP + tl)
      double2 c[N];
      const double2* Wb = W + (size_t)buf * n + (size_t)(rank * NP + tl) * N + tx;
#pragma unroll
      for (int z = 0; z < N; ++z) c[z] = __ldcg(Wb + (size_t)z * N * N);
      fft<N, -1>(c);
      double2* fh = fhat + tl * N * N + tx;
#pragma unroll
      for (int lz = 0; lz < N; ++lz) fh[lz * N] = c[lz];
    }
    buf ^= 1;

    // ---- a5/a6: A gain directions + the loss ---------------------------------------------
    double gacc[N];
#pragma unroll
    for (int y = 0; y < N; ++y) gacc[y] = 0.0;
#pragma unroll 1
    for (int d = 0; d <= p.A; ++d) {
      mbar_wait(mbar, tphase);
      tphase ^= 1;
      {
        double2 x[N];
        const double2* fh = fhat + tl * N * N + tx;
        const double2* tb = tbuf + tl * N * N + tx;
#pragma unroll
        for (int lz = 0; lz < N; ++lz) {
          const double2 T = tb[lz * N], F = fh[lz * N];
          x[lz] = make_double2(fma(T.x, F.x, -T.y * F.y), fma(T.x, F.y, T.y * F.x));
        }
        fft<N, +1>(x);
        double2* Wb = W + (size_t)buf * n + (size_t)(rank * NP + tl) * N + tx;
#pragma unroll
        for (int jz = 0; jz < N; ++jz) Wb[(size_t)jz * N * N] = x[jz];
      }
      __syncthreads();  // tbuf consumed
      if (t == 0 && d < p.A) load_table_slab<N, P>(tbuf, p.tables, d + 1, rank, mbar);
      cluster_sync_all();
      {
        const double2* Wp = W + (size_t)buf * n + (size_t)rank * C::SLAB;
        for (int e = t; e < C::SLAB; e += C::THREADS) {
          const int x = e % N, yz = e / N;
          pln[yz * RS + x] = __ldcg(Wp + e);
        }
      }
      __syncthreads();
      {
        double2 r[N];
        double2* row = pln + tl * N * RS + tx * RS;
#pragma unroll
        for (int x = 0; x < N; ++x) r[x] = row[x];
        fft<N, +1>(r);
#pragma unroll
        for (int x = 0; x < N; ++x) row[x] = r[x];
      }
      __syncthreads();
      {
        double2 c[N];
        const double2* col = pln + tl * N * RS + tx;
#pragma unroll
        for (int y = 0; y < N; ++y) c[y] = col[y * RS];
        fft<N, +1>(c);
        if (d < p.A) {
#pragma unroll
          for (int y = 0; y < N; ++y) gacc[y] = fma(c[y].x, c[y].y, gacc[y]);
        } else {
          const int z = rank * NP + tl;
          double* g = G + tl * N * N + tx;
#pragma unroll
          for (int y = 0; y < N; ++y) {
            const double fs = gather_fstar(p.f_in, p.tp, cell, tx + N * (y + N * z), tx, y, z, n);
            g[y * N] = gacc[y] - fs * c[y].x;
          }
        }
      }
      buf ^= 1;
    }

    // ---- a8 + a9: projection and Euler (or write Q) ---------------------------------------
    const int z = rank * NP + tl;
    const double* g = G + tl * N * N + tx;
    double* out = p.f_out + cell * (int64_t)n;
    if (p.mode == 0) {
#pragma unroll 4
      for (int y = 0; y < N; ++y) out[tx + N * (y + N * z)] = g[y * N];
    } else {
      double lam[5] = {0, 0, 0, 0, 0};
      if (p.project) {
        const double vx = node_v(tx, p.L, p.dv), vz = node_v(z, p.L, p.dv);
        double m[5] = {0, 0, 0, 0, 0};
        for (int y = 0; y < N; ++y) {
          const double q = g[y * N], vy = node_v(y, p.L, p.dv);
          m[0] += q;
          m[1] += vx * q;
          m[2] += vy * q;
          m[3] += vz * q;
          m[4] += (vx * vx + vy * vy + vz * vz) * q;
        }
#pragma unroll
        for (int c = 0; c < 5; ++c) {
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
        }
        // warps -> CTA partial (fixed order), then the cluster sum through DSMEM in rank order
        __syncthreads();
        constexpr int NW = (C::THREADS + 31) / 32;
        double* wpart = reinterpret_cast<double*>(pln);  // scratch: [NW][5]
        if ((t & 31) == 0) {
#pragma unroll
          for (int c = 0; c < 5; ++c) wpart[(t >> 5) * 5 + c] = m[c];
        }
        __syncthreads();
        if (t < 5) {
          double s = 0.0;
          for (int w = 0; w < NW; ++w) s += wpart[w * 5 + t];
          part[t] = s;
        }
        cluster_sync_all();
        double mu[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) mu[c] = 0.0;
        for (int r = 0; r < P; ++r) {
          const double* rp = cluster.map_shared_rank(part, r);
#pragma unroll
          for (int c = 0; c < 5; ++c) mu[c] += rp[c];
        }
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < 5; ++b) s = fma(p.Ginv[a * 5 + b], mu[b], s);
          lam[a] = s;
        }
      }
      const double vx = node_v(tx, p.L, p.dv), vz = node_v(z, p.L, p.dv);
      bool bad = false;
      for (int y = 0; y < N; ++y) {
        const double vy = node_v(y, p.L, p.dv);
        const int k = tx + N * (y + N * z);
        const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * vz + lam[4] * (vx * vx + vy * vy + vz * vz);
        const double fs = gather_fstar(p.f_in, p.tp, cell, k, tx, y, z, n);
        const double o = fma(p.dt_tau, g[y * N] - corr, fs);
        bad |= !isfinite(o);
        out[k] = o;
      }
      if (bad) atomicOr(p.nonfinite, 1);
      if (p.project) cluster_sync_all();  // part[] is read remotely before it is rewritten
    }
  }
}

template <int N>
static cudaError_t launch3(const StepParams& p, int nclusters, cudaStream_t s) {
  constexpr int P = 8;
  using C = Cfg3<N, P>;
  auto kern = k_step3d<N, P>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * P);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int N>
static int max_clusters3() {
  constexpr int P = 8;
  using C = Cfg3<N, P>;
  auto kern = k_step3d<N, P>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P * 64);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) return 0;
  return ncl;
}

cudaError_t launch_step3d(int N, const StepParams& p, int nclusters, cudaStream_t s) {
  switch (N) {
    case 8: return launch3<8>(p, nclusters, s);
    case 16: return launch3<16>(p, nclusters, s);
    case 32: return launch3<32>(p, nclusters, s);
    default: return cudaErrorInvalidValue;
  }
}

int max_active_clusters3d(int N) {
  switch (N) {
    case 8: return max_clusters3<8>();
    case 16: return max_clusters3<16>();
    case 32: return max_clusters3<32>();
    default: return 0;
  }
}

size_t scratch_elems3d(int N) { return (size_t)2 * N * N * N; }

}  // namespace fks
