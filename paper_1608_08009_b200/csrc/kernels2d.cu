// 2D fused collision / step kernel (a3-a9) for Maxwell molecules on an N^2 velocity grid.
//
// A group of N threads owns one cell (256 / N groups per CTA, persistent over cells).
//   f^ lives in tensor memory: thread l_x keeps its column f^(l_x, .) in its TMEM lane (4N
//   32-bit columns; the two warps sharing a lane quarter use disjoint column ranges), written by
//   tcgen05.st after the forward transform and read back by tcgen05.ld for every direction.
//   One N x N work plane per cell in SMEM (XOR-swizzled: element (r, c) at r*N + (c ^ (r & 7)),
//   conflict-free for row and column sweeps).
//   The tables are even, T(-l) = T(l) (reading #10), so the CTA keeps only the columns
//   l_x = 0..N/2 of every direction in SMEM, loaded once per CTA (78 KB at N = 32, A = 8); a
//   direction set too large for that reads the full tables from L2 instead (TAB_SMEM = false).
// Per direction p:
//   column pass: thread l_x forms X = (alpha~_p + i alpha'~_p) f^ along l_y and IFFTs it,
//   row pass:    thread j_y IFFTs its row and accumulates G[j_y][.] += Re z Im z in registers.
// The loss is the (A+1)-th direction with table (D~, 0).  Thread j_y then owns row j_y of Q for
// the projection (a group reduction of 4 moments) and the Euler update.
// Folded tables: T[p][l_y][l_x] double2 = (s w_p alpha_p / n, alpha'_p / n); T[A] = (s D / n, 0).
#include <cstdlib>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace fks {

template <int N>
struct Cfg2 {
  static constexpr int THREADS = 256;
  static constexpr int GROUPS = THREADS / N;  // cells in flight per CTA
  static constexpr int HC = N / 2 + 1;        // stored table columns l_x = 0..N/2
  static constexpr size_t PER_GROUP = (size_t)N * N * 16;
  static constexpr size_t OFF_DELTA = GROUPS * PER_GROUP;
  static constexpr size_t OFF_TMEM = OFF_DELTA + 3 * kMaxN + 8;  // 8-byte aligned slot
  static constexpr size_t OFF_TAB = (OFF_TMEM + 4 + 127) / 128 * 128;
  static constexpr int FCOLS = 4 * N;                          // TMEM columns per thread: f^ column
  // f* row cache (N >= 16): row j_y = tx of f* (N fp64 = 2N columns), read back by the loss
  // term and the Euler update instead of re-gathering f from global memory.
  static constexpr bool FS_TMEM = N >= 16;
  static constexpr int SCOLS = FS_TMEM ? 2 * N : 0;
  static constexpr int USED_COLS = (THREADS / 128) * (FCOLS + SCOLS);
  static constexpr int TMEM_COLS = USED_COLS <= 32 ? 32 : USED_COLS <= 64 ? 64 : USED_COLS <= 128 ? 128
                                 : USED_COLS <= 256 ? 256 : 512;
  static size_t smem(int A, bool tab_smem) {
    return OFF_TAB + (tab_smem ? (size_t)(A + 1) * N * HC * 16 : 0);
  }
  static_assert(TMEM_COLS >= 32 && (TMEM_COLS & (TMEM_COLS - 1)) == 0, "TMEM allocation: power of two >= 32");
};

__device__ __forceinline__ int swz2(int r, int c) { return c ^ (r & 7); }

template <int N>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = N / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(mask, v, o, N);
  return v;
}

__device__ __forceinline__ uint32_t smem_addr2(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tmem2_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem2_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

template <int N, bool TAB_SMEM>
__global__ void __launch_bounds__(Cfg2<N>::THREADS, 1) k_step2d(const StepParams p) {
  using C = Cfg2<N>;
  constexpr int n = N * N;
  constexpr int HC = C::HC;
  extern __shared__ __align__(128) unsigned char smem[];
  const int g = threadIdx.x / N;  // group (cell slot) of this thread
  const int tx = threadIdx.x % N;
  double2* wk = reinterpret_cast<double2*>(smem + g * C::PER_GROUP);  // [y][x], swizzled
  const unsigned lane = threadIdx.x & 31;
  const unsigned mask = N >= 32 ? 0xffffffffu : (((1u << N) - 1u) << (lane & ~(unsigned)(N - 1)));
  // cells are walked warp by warp (32/N cells per warp) so every lane of a warp executes the
  // warp-collective tcgen05 instructions; a group past the end recomputes the last cell and
  // skips its stores.
  constexpr int CPW = 32 / N < 1 ? 1 : 32 / N;
  const int stride = gridDim.x * C::GROUPS;
  int8_t (*sdelta)[kMaxN] = reinterpret_cast<int8_t (*)[kMaxN]>(smem + C::OFF_DELTA);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  double2* tab = reinterpret_cast<double2*>(smem + C::OFF_TAB);  // [A+1][l_y][HC]
  load_delta(p.tp, sdelta);
  if (TAB_SMEM) {
    const int tot = (p.A + 1) * N * HC;
    FKS_CHECK((int64_t)(p.A + 1) * n <= p.table_elems);
    for (int e = threadIdx.x; e < tot; e += C::THREADS) {
      const int c = e % HC, ly = (e / HC) % N, d = e / (HC * N);
      tab[e] = __ldg(p.tables + (size_t)d * n + ly * N + c);
    }
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr2(tmem_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = *tmem_slot;
  const int w = threadIdx.x >> 5;
  const uint32_t taddr = tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * C::FCOLS);
  // f* row cache of this thread (FS_TMEM)
  const uint32_t saddr = tbase + ((uint32_t)(32 * (w & 3)) << 16) +
                         (uint32_t)((C::THREADS / 128) * C::FCOLS + (w >> 2) * C::SCOLS);
  // f*(x, j_y = tx) for x in [16 ch, 16 ch + 16): from the TMEM row cache
  auto fs_chunk = [&](int ch, double (&fs)[16]) {
    uint32_t v[32];
    tmem2_ld32(saddr + ch * 32, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) fs[i] = __hiloint2double(v[2 * i + 1], v[2 * i]);
  };

  for (int base = blockIdx.x * C::GROUPS + (threadIdx.x >> 5) * CPW; base < p.ncells; base += stride) {
    const int itr = base + ((threadIdx.x & 31) / N) % CPW;
    const bool active = itr < p.ncells;
    const int it = active ? itr : p.ncells - 1;
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc = cell_coord(p.tp, cell);
    // the next cell of this group (homogeneous case: a contiguous 8 KB row block) -> L2
    if (p.tp.dx == 0 && tx == 0 && !p.cell_list) {
      const int nx = itr + stride;
      if (nx < p.ncells)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p.f_in + (int64_t)nx * n),
                     "r"((uint32_t)(n * sizeof(double)))
                     : "memory");
    }
    // a3: row y = tx of f*, forward FFT along x
    {
      double2 r[N];
#pragma unroll
      for (int x = 0; x < N; ++x) r[x].y = 0.0;
      if (p.tp.dx == 0) {  // the row is contiguous: 16-byte loads, all in flight at once
        const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * (int64_t)n + N * tx);
#pragma unroll
        for (int x = 0; x < N / 2; ++x) {
          const double2 v = __ldg(src + x);
          r[2 * x].x = v.x;
          r[2 * x + 1].x = v.y;
        }
      } else {
#pragma unroll
        for (int x = 0; x < N; ++x) r[x].x = gather_fstar(p.f_in, p.tp, cc, x + N * tx, x, tx, 0, n, sdelta);
      }
      if constexpr (C::FS_TMEM) {
#pragma unroll
        for (int ch = 0; ch < N / 16; ++ch) {
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            v[2 * i] = __double2loint(r[ch * 16 + i].x);
            v[2 * i + 1] = __double2hiint(r[ch * 16 + i].x);
          }
          tmem2_st32(saddr + ch * 32, v);
        }
      }
      fft<N, -1>(r);
#pragma unroll
      for (int x = 0; x < N; ++x) wk[tx * N + swz2(tx, x)] = r[x];
    }
    __syncwarp(mask);
    {  // column l_x = tx, forward FFT along y, f^ column -> this thread's TMEM columns
      double2 c[N];
#pragma unroll
      for (int y = 0; y < N; ++y) c[y] = wk[y * N + swz2(y, tx)];
      fft<N, -1>(c);
#pragma unroll
      for (int ch = 0; ch < N / 8; ++ch) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[4 * i + 0] = __double2loint(c[ch * 8 + i].x);
          v[4 * i + 1] = __double2hiint(c[ch * 8 + i].x);
          v[4 * i + 2] = __double2loint(c[ch * 8 + i].y);
          v[4 * i + 3] = __double2hiint(c[ch * 8 + i].y);
        }
        tmem2_st32(taddr + ch * 32, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    __syncwarp(mask);
    double gacc[N];
#pragma unroll
    for (int x = 0; x < N; ++x) gacc[x] = 0.0;
    const bool neg = tx > N / 2;  // column l_x > N/2 reads the table at (-l_x, -l_y)
    const int tcol = neg ? N - tx : tx;
#pragma unroll 1
    for (int d = 0; d <= p.A; ++d) {
      // pass 0: column l_x = tx, X = T f^ from TMEM, IFFT along y -> work plane;
      // pass 1: row j_y = tx from the work plane, IFFT along x, accumulate.  One FFT body for
      // both passes halves the loop's instruction footprint (instruction-cache misses were the
      // top stall reason of the two-body loop, profiles/r01_ncu_k_step2d.json).
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        double2 c[N];
        if (pass == 0) {
#pragma unroll
          for (int ch = 0; ch < N / 8; ++ch) {
            // table entries first: their shared-memory latency overlaps the TMEM load's
            double2 tt[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int ly = ch * 8 + i;
              if (TAB_SMEM) {
                const int row = neg ? (N - ly) & (N - 1) : ly;
                tt[i] = tab[((size_t)d * N + row) * HC + tcol];
              } else {
                FKS_CHECK((int64_t)d * n + ly * N + tx < p.table_elems);
                tt[i] = __ldg(p.tables + (size_t)d * n + ly * N + tx);
              }
            }
            uint32_t v[32];
            tmem2_ld32(taddr + ch * 32, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int ly = ch * 8 + i;
              const double2 t = tt[i];
              const double Fx = __hiloint2double(v[4 * i + 1], v[4 * i + 0]);
              const double Fy = __hiloint2double(v[4 * i + 3], v[4 * i + 2]);
              c[ly] = make_double2(fma(t.x, Fx, -t.y * Fy), fma(t.x, Fy, t.y * Fx));
            }
          }
        } else {
#pragma unroll
          for (int x = 0; x < N; ++x) c[x] = wk[tx * N + swz2(tx, x)];
        }
        fft<N, +1>(c);
        if (pass == 0) {
#pragma unroll
          for (int y = 0; y < N; ++y) wk[y * N + swz2(y, tx)] = c[y];
        } else if (d < p.A) {
#pragma unroll
          for (int x = 0; x < N; ++x) gacc[x] = fma(c[x].x, c[x].y, gacc[x]);
        } else if constexpr (C::FS_TMEM) {
#pragma unroll
          for (int ch = 0; ch < N / 16; ++ch) {
            double fs[16];
            fs_chunk(ch, fs);
#pragma unroll
            for (int i = 0; i < 16; ++i) gacc[ch * 16 + i] = gacc[ch * 16 + i] - fs[i] * c[ch * 16 + i].x;
          }  // gacc now holds Q
        } else {
#pragma unroll
          for (int x = 0; x < N; ++x) {
            const double fs = gather_fstar(p.f_in, p.tp, cc, x + N * tx, x, tx, 0, n, sdelta);
            gacc[x] = gacc[x] - fs * c[x].x;  // gacc now holds Q
          }
        }
        __syncwarp(mask);
      }
    }
    double* out = p.f_out + cell * (int64_t)n;
    const double* q = gacc;
    if (p.mode == 0) {
      if (active) {
#pragma unroll
        for (int x = 0; x < N; ++x) out[x + N * tx] = q[x];
      }
      continue;
    }
    double lam[4] = {0, 0, 0, 0};
    const double vy = node_v(tx, p.L, p.dv);
    if (p.project) {
      double m[4] = {0, 0, 0, 0};
#pragma unroll
      for (int x = 0; x < N; ++x) {
        const double vx = node_v(x, p.L, p.dv);
        m[0] += q[x];
        m[1] += vx * q[x];
        m[2] += vy * q[x];
        m[3] += (vx * vx + vy * vy) * q[x];
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) m[c] = group_sum<N>(m[c], mask);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) s = fma(p.Ginv[a * 4 + b], m[b], s);
        lam[a] = s;
      }
    }
    bool bad = false;
    const double* hbase = p.mode == 2 ? p.f_base + cell * (int64_t)n : nullptr;
    auto euler = [&](int x, double fs) {
      const double vx = node_v(x, p.L, p.dv);
      const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * (vx * vx + vy * vy);
      double o = fma(p.dt_tau, q[x] - corr, fs);
      if (hbase) o = 0.5 * (o + __ldcs(hbase + x + N * tx));  // Heun: (f* + E(f1)) / 2 (NEXT-4)
      bad |= !isfinite(o);
      if (active) out[x + N * tx] = o;
    };
    if constexpr (C::FS_TMEM) {
#pragma unroll
      for (int ch = 0; ch < N / 16; ++ch) {
        double fs[16];
        fs_chunk(ch, fs);
#pragma unroll
        for (int i = 0; i < 16; ++i) euler(ch * 16 + i, fs[i]);
      }
    } else {
#pragma unroll
      for (int x = 0; x < N; ++x) euler(x, gather_fstar(p.f_in, p.tp, cc, x + N * tx, x, tx, 0, n, sdelta));
    }
    if (bad && active) atomicOr(p.nonfinite, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(C::TMEM_COLS) : "memory");
}

template <int N>
static cudaError_t launch2(const StepParams& p, int nblocks, cudaStream_t s) {
  using C = Cfg2<N>;
  const bool tab_smem = C::smem(p.A, true) <= 232448;
  const size_t sm = C::smem(p.A, tab_smem);
  auto kern = tab_smem ? k_step2d<N, true> : k_step2d<N, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  kern<<<nblocks, C::THREADS, sm, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_step2d(int N, const StepParams& p, int nblocks, cudaStream_t s) {
  switch (N) {
    case 8: return launch2<8>(p, nblocks, s);
    case 16: return launch2<16>(p, nblocks, s);
    case 32: return launch2<32>(p, nblocks, s);
    default: return cudaErrorInvalidValue;
  }
}

int cells_per_block2d(int N) {
  switch (N) {
    case 8: return Cfg2<8>::GROUPS;
    case 16: return Cfg2<16>::GROUPS;
    case 32: return Cfg2<32>::GROUPS;
    default: return 0;
  }
}

bool use_pair2d(int N, int A) {
  if (N == 64) return true;
  if (N != 32 || !step2d_pair_fits(N, A)) return false;
  static const bool knob = [] {  // development knob, read once
    const char* e = getenv("FKS_2D_PAIR");
    return e && atoi(e) == 1;
  }();
  return knob;
}

}  // namespace fks
