// 3D fused collision / step kernel (a3-a9) for hard spheres on an N^3 velocity grid.
//
// One thread-block cluster of P CTAs owns one cell at a time (persistent over cells).  The
// cell's N^3 spectrum does not fit one SM (N = 32: 512 KiB per complex transform), so the
// 3D inverse FFT of each direction is split by planes:
//   CTA r owns the spectrum planes l_y in [r N/P, (r+1) N/P)  (f^ resident in SMEM) and
//   the output planes  j_z in [r N/P, (r+1) N/P)             (gain accumulator in registers).
// Per direction p the CTA
//   z: forms X = (alpha~_p + i alpha'~_p) f^ on its pencils and IFFTs along z in registers,
//      then writes the pencils to a per-cluster L2 exchange buffer (the transpose);
//   xy: after a cluster barrier, bulk-copies its own j_z planes back (cp.async.bulk, async
//      proxy), IFFTs along x and y and accumulates G += Re z * Im z -- two real transforms
//      packed in one complex IFFT, exact because the symmetrised tables are real and even
//      (reading #10).
// Software pipeline (per cell, d = 0..A, the loss is d = A with table (D~, 0)):
//   z(0); arrive(0);
//   for d: wait(d); bulk W(d) -> SMEM; z(d+1) [overlaps the copy]; xy(d); arrive(d+1)
// so the exchange latency hides behind z(d+1) and the release fence of arrive(d+1) finds the
// z(d+1) stores long completed.  The exchange goes through L2 (measured ~15 TB/s) rather than
// DSMEM (measured ~2 TB/s, profiles/r01_microbench.txt).  The next direction's table slab is
// prefetched with cp.async.bulk while xy runs.  Epilogue: Q = G - f* Re z(loss),
// projection to zero moments (5-sum cluster reduction through DSMEM) and
// F^{n+1} = f* + (dt/tau) Pi Q, or Q in collide mode.
// Tables are pre-folded on the host: alpha~ = s w_p alpha_p / n, alpha'~ = alpha'_p / n,
// D~ = s D / n (s = Btilde kappa^-(d+gamma)); layout T[p][l_y][l_z][l_x] as double2.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace fks {

template <int N, int P>
struct Cfg3 {
  static constexpr int NP = N / P;        // planes per CTA
  static constexpr int THREADS = N * NP;  // one pencil / row / column per thread
  static constexpr int RS = N + 1;        // padded row stride (bank-conflict-free rows and columns)
  static constexpr int SLAB = NP * N * N;     // complex elements of f^ / table slab
  static constexpr int PSLAB = NP * N * RS;   // complex elements of a padded plane slab
  static constexpr int WPLANE = N * RS;       // padded plane in the exchange buffer
  static constexpr size_t WBUF = (size_t)N * WPLANE;  // one exchange buffer (all N j_z planes)
  static constexpr int NBUF = 2;
  static constexpr size_t OFF_FHAT = 0;  // f^ slab; reused as G/Q after the last z-pass
  static constexpr size_t OFF_TBUF = OFF_FHAT + (size_t)SLAB * 16;
  static constexpr size_t OFF_PLN = OFF_TBUF + (size_t)SLAB * 16;
  static constexpr size_t OFF_MBAR = OFF_PLN + (size_t)PSLAB * 16;
  static constexpr size_t OFF_PART = OFF_MBAR + 16;
  static constexpr size_t SMEM = OFF_PART + 8 * 8;
  static_assert((size_t)NP * N * N * 8 <= (size_t)SLAB * 16, "G must fit in the f^ slab");
};

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() { cl_arrive(); cl_wait(); }

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

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  constexpr uint32_t chunk = 32768;
  mbar_expect_tx(bar, bytes);
  for (uint32_t off = 0; off < bytes; off += chunk)
    bulk_g2s(reinterpret_cast<char*>(dst) + off, reinterpret_cast<const char*>(src) + off,
             bytes - off < chunk ? bytes - off : chunk, bar);
}

// One pencil (l_x = tx, local l_y = tl) of direction d: X = T (x) f^, IFFT along z, store to W.
template <int N, int P>
__device__ __forceinline__ void zpass(const double2* fhat, const double2* tbuf, double2* Wb, int rank, int tx,
                                      int tl) {
  using C = Cfg3<N, P>;
  double2 x[N];
  const double2* fh = fhat + tl * N * N + tx;
  const double2* tb = tbuf + tl * N * N + tx;
#pragma unroll
  for (int lz = 0; lz < N; ++lz) {
    const double2 T = tb[lz * N], F = fh[lz * N];
    x[lz] = make_double2(fma(T.x, F.x, -T.y * F.y), fma(T.x, F.y, T.y * F.x));
  }
  fft<N, +1>(x);
  double2* w = Wb + (size_t)(rank * C::NP + tl) * C::RS + tx;
#pragma unroll
  for (int jz = 0; jz < N; ++jz) w[(size_t)jz * C::WPLANE] = x[jz];
}

template <int N, int P>
__global__ void __launch_bounds__(Cfg3<N, P>::THREADS, 1) k_step3d(const StepParams p) {
  using C = Cfg3<N, P>;
  constexpr int NP = C::NP, RS = C::RS;
  constexpr int n = N * N * N;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* fhat = reinterpret_cast<double2*>(smem + C::OFF_FHAT);  // [NP l_y][N l_z][N l_x]
  double* G = reinterpret_cast<double*>(smem + C::OFF_FHAT);       // [NP j_z][N j_y][N j_x] (after z(A))
  double2* tbuf = reinterpret_cast<double2*>(smem + C::OFF_TBUF);  // [NP l_y][N l_z][N l_x]
  double2* pln = reinterpret_cast<double2*>(smem + C::OFF_PLN);    // [NP j_z][N y][RS x]
  uint64_t* tbar = reinterpret_cast<uint64_t*>(smem + C::OFF_MBAR);
  uint64_t* wbar = tbar + 1;
  double* part = reinterpret_cast<double*>(smem + C::OFF_PART);

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / P;
  const int ncl = gridDim.x / P;
  const int t = threadIdx.x;
  const int tx = t % N;  // l_x / j_x / row index along the fast axis
  const int tl = t / N;  // local plane index
  double2* Wbase = p.scratch + (size_t)cid * C::NBUF * C::WBUF;  // [NBUF][N j_z][N l_y][RS l_x]
  constexpr uint32_t kTabBytes = C::SLAB * 16;
  constexpr uint32_t kPlaneBytes = C::PSLAB * 16;

  if (t == 0) {
    mbar_init(tbar, 1);
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t tphase = 0, wphase = 0;
  int buf = 0;

  for (int it = cid; it < p.ncells; it += ncl) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    if (t == 0)
      bulk_load(tbuf, p.tables + (size_t)rank * C::SLAB, kTabBytes, tbar);

    // ---- a3 + a4: gather f* (own j_z planes) and forward FFT in x, y, then z -------------
    {
      constexpr int PER = NP * N * N / C::THREADS;  // = N: elements per thread
      constexpr int B = PER < 16 ? PER : 16;        // loads in flight per batch
#pragma unroll 1
      for (int b0 = 0; b0 < PER; b0 += B) {
        double v[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int e = t + (b0 + j) * C::THREADS;
          const int x = e % N, y = (e / N) % N, z = rank * NP + e / (N * N);
          v[j] = gather_fstar(p.f_in, p.tp, cell, x + N * (y + N * z), x, y, z, n);
        }
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int e = t + (b0 + j) * C::THREADS;
          const int x = e % N, y = (e / N) % N, zl = e / (N * N);
          pln[zl * N * RS + y * RS + x] = make_double2(v[j], 0.0);
        }
      }
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
      double2* Wb = Wbase + (size_t)buf * C::WBUF + (size_t)(rank * NP + tl) * C::WPLANE + tx;
#pragma unroll
      for (int ly = 0; ly < N; ++ly) Wb[ly * RS] = c[ly];
    }
    cluster_sync_all();
    {
      double2 c[N];
      const double2* Wb = Wbase + (size_t)buf * C::WBUF + (size_t)(rank * NP + tl) * RS + tx;
#pragma unroll
      for (int z = 0; z < N; ++z) c[z] = __ldcg(Wb + (size_t)z * C::WPLANE);
      fft<N, -1>(c);
      double2* fh = fhat + tl * N * N + tx;
#pragma unroll
      for (int lz = 0; lz < N; ++lz) fh[lz * N] = c[lz];
    }
    buf ^= 1;
    __syncthreads();  // f^ complete

    // ---- a5/a6: A gain directions + the loss, software-pipelined --------------------------
    mbar_wait(tbar, tphase);
    tphase ^= 1;
    zpass<N, P>(fhat, tbuf, Wbase + (size_t)buf * C::WBUF, rank, tx, tl);
    __syncthreads();
    if (t == 0) bulk_load(tbuf, p.tables + (size_t)1 * n + (size_t)rank * C::SLAB, kTabBytes, tbar);
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    cl_arrive();

    double gacc[N];
#pragma unroll
    for (int y = 0; y < N; ++y) gacc[y] = 0.0;
#pragma unroll 1
    for (int d = 0; d <= p.A; ++d) {
      const int bd = buf;  // exchange buffer of direction d
      cl_wait();           // W(d) complete cluster-wide; W(d-1) no longer read anywhere
      if (t == 0) {
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        bulk_load(pln, Wbase + (size_t)bd * C::WBUF + (size_t)rank * C::PSLAB, kPlaneBytes, wbar);
      }
      if (d < p.A) {
        mbar_wait(tbar, tphase);
        tphase ^= 1;
        zpass<N, P>(fhat, tbuf, Wbase + (size_t)(bd ^ 1) * C::WBUF, rank, tx, tl);
        __syncthreads();  // tbuf consumed
        if (t == 0 && d + 2 <= p.A)
          bulk_load(tbuf, p.tables + (size_t)(d + 2) * n + (size_t)rank * C::SLAB, kTabBytes, tbar);
      }
      mbar_wait(wbar, wphase);
      wphase ^= 1;
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
        __syncthreads();  // pln free for the next bulk copy
        fft<N, +1>(c);
        if (d < p.A) {
#pragma unroll
          for (int y = 0; y < N; ++y) gacc[y] = fma(c[y].x, c[y].y, gacc[y]);
        } else {
          const int z = rank * NP + tl;
          double* g = G + tl * N * N + tx;
          double fs[N];
#pragma unroll
          for (int y = 0; y < N; ++y) fs[y] = gather_fstar(p.f_in, p.tp, cell, tx + N * (y + N * z), tx, y, z, n);
#pragma unroll
          for (int y = 0; y < N; ++y) {
            g[y * N] = gacc[y] - fs[y] * c[y].x;
            gacc[y] = fs[y];  // gacc now holds the f* column for the Euler update
          }
        }
      }
      buf ^= 1;
      if (d < p.A) {
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        cl_arrive();  // z(d+1) stores (issued before xy(d)) are complete by now
      }
    }
    __syncthreads();

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
        constexpr int W = C::THREADS < 32 ? C::THREADS : 32;
        constexpr unsigned mask = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
#pragma unroll
        for (int c = 0; c < 5; ++c) {
#pragma unroll
          for (int o = W / 2; o >= 1; o >>= 1) m[c] += __shfl_xor_sync(mask, m[c], o);
        }
        // warps -> CTA partial (fixed order), then the cluster sum through DSMEM in rank order
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
#pragma unroll
      for (int y = 0; y < N; ++y) {
        const double vy = node_v(y, p.L, p.dv);
        const int k = tx + N * (y + N * z);
        const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * vz + lam[4] * (vx * vx + vy * vy + vz * vz);
        const double o = fma(p.dt_tau, g[y * N] - corr, gacc[y]);
        bad |= !isfinite(o);
        out[k] = o;
      }
      if (bad) atomicOr(p.nonfinite, 1);
      if (p.project) {  // part[] is read remotely before it is rewritten (or the CTA exits);
        // the remote loads completed (their values were consumed), so no release is needed
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
        cl_wait();
      }
    }
    __syncthreads();  // G (= f^ slab) consumed before the next cell's f^
  }
}

template <int N, int P>
static cudaLaunchConfig_t make_cfg(int nclusters, cudaStream_t s, cudaLaunchAttribute* attr) {
  using C = Cfg3<N, P>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * P);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

template <int N, int P>
static cudaError_t prep() {
  using C = Cfg3<N, P>;
  auto kern = k_step3d<N, P>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) return e;
  if (P > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

template <int N, int P>
static cudaError_t launch3(const StepParams& p, int nclusters, cudaStream_t s) {
  cudaError_t e = prep<N, P>();
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = make_cfg<N, P>(nclusters, s, attr);
  return cudaLaunchKernelEx(&cfg, k_step3d<N, P>, p);
}

template <int N, int P>
static int max_clusters3() {
  if (prep<N, P>() != cudaSuccess) return 0;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = make_cfg<N, P>(64, 0, attr);
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, k_step3d<N, P>, &cfg) != cudaSuccess) return 0;
  return ncl;
}

// CTAs per cell for N = 32 (8 or 16); 8 for the small grids.  FKS_P32 env var overrides (tuning).
static int p32() {
  static int v = [] {
    const char* e = getenv("FKS_P32");
    return (e && atoi(e) == 16) ? 16 : 8;
  }();
  return v;
}

cudaError_t launch_step3d(int N, const StepParams& p, int nclusters, cudaStream_t s) {
  switch (N) {
    case 8: return launch3<8, 8>(p, nclusters, s);
    case 16: return launch3<16, 8>(p, nclusters, s);
    case 32: return p32() == 16 ? launch3<32, 16>(p, nclusters, s) : launch3<32, 8>(p, nclusters, s);
    default: return cudaErrorInvalidValue;
  }
}

int max_active_clusters3d(int N) {
  switch (N) {
    case 8: return max_clusters3<8, 8>();
    case 16: return max_clusters3<16, 8>();
    case 32: return p32() == 16 ? max_clusters3<32, 16>() : max_clusters3<32, 8>();
    default: return 0;
  }
}

size_t scratch_elems3d(int N) { return (size_t)Cfg3<32, 8>::NBUF * N * N * (N + 1); }

}  // namespace fks
