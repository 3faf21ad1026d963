// 2D fused collision / step kernel (a3-a9) with every N-point pencil split over a lane pair
// (N = 64, and N = 32 as the higher-occupancy alternative to kernels2d.cu).
//
// Same method as kernels2d.cu (per direction a packed complex IFFT (alpha~ + i alpha'~) f^,
// G += Re z Im z; the loss as the (A+1)-th item; projection; Euler), but each pencil lives in two
// threads (h = lane & 1 owns N/2 complex values) with one radix-2 stage across the pair through
// shuffles:
//   forward (DIF): thread h holds x[N/2 h + j] (halves) -> thread h gets X[2m + h] (parity);
//   inverse (DIT): thread h holds x[2m + h] (parity) -> thread h gets X[N/2 h + j] (halves);
// the N/2-point remainders are the register FFTs of fft.cuh.  The layouts chain without reshuffles:
// forward rows (halves of f*) -> SMEM -> forward columns (halves) -> f^ in TMEM in parity order ->
// per direction the column IFFT (parity in, halves out) -> SMEM -> the row IFFT reads its parity
// inputs from SMEM and leaves thread (row q, half h) the outputs j_x in [N/2 h, N/2 h + N/2), which
// is exactly the f* half it cached in TMEM during the forward pass.
// Half the registers per thread buys twice the warps per SM: N = 64 needs it to fit at all (a
// 64-point pencil next to its accumulator exceeds 255 registers); N = 32 runs 16 warps per SM
// instead of 8.  One N x N work plane per cell in SMEM (XOR swizzle c ^ ((r & 3) << 1): conflict-free
// for the column sweeps and the strided row reads).  Tables: N = 32 keeps the even half (columns
// l_x = 0..N/2, reading #10) of every direction in SMEM; N = 64 reads them from L2.
#include "common.cuh"
#include "fft.cuh"
#include "fftp.cuh"
#include "kernels.cuh"

namespace fks {

namespace {

template <int N>
struct CfgP {
  static constexpr int H = N / 2;                   // complex values per thread of a pencil
  static constexpr int THREADS = N == 64 ? 256 : 512;
  static constexpr int GT = 2 * N;                  // threads per cell
  static constexpr int CELLS = THREADS / GT;        // cells per CTA
  static constexpr int NWG = GT / 32;               // warps per cell
  static constexpr bool TAB_SMEM = N <= 32;
  static constexpr int HC = N / 2 + 1;              // stored table columns (TAB_SMEM)
  static constexpr size_t PLANE = (size_t)N * N * 16;
  static constexpr int FCOLS = 4 * H;               // f^ half column in TMEM (H complex fp64)
  static constexpr int SCOLS = 2 * H;               // f* half row (H fp64)
  static constexpr int WPQ = THREADS / 128;         // warps sharing a TMEM lane quarter
  static_assert(WPQ * (FCOLS + SCOLS) <= 512, "TMEM columns");
  static constexpr size_t OFF_DELTA = CELLS * PLANE;
  static constexpr size_t OFF_RED = OFF_DELTA + 3 * kMaxN;  // [CELLS][NWG][4]
  static constexpr size_t OFF_TMEM = (OFF_RED + CELLS * NWG * 4 * 8 + 15) / 16 * 16;
  static constexpr size_t OFF_TAB = (OFF_TMEM + 16 + 127) / 128 * 128;
  static size_t smem(int A) { return OFF_TAB + (TAB_SMEM ? (size_t)(A + 1) * N * HC * 16 : 0); }
};

template <int N>
__device__ __forceinline__ int swp(int r, int c) { return r * N + (c ^ ((r & 3) << 1)); }

__device__ __forceinline__ void tmem_st32p(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld32p(uint32_t taddr, uint32_t (&v)[32]) {
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

__device__ __forceinline__ void grp_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

}  // namespace

template <int N>
__global__ void __launch_bounds__(CfgP<N>::THREADS, 1) k_step2dp(const StepParams p) {
  using C = CfgP<N>;
  constexpr int n = N * N, H = C::H, GT = C::GT;
  extern __shared__ __align__(128) unsigned char smem[];
  const int g = threadIdx.x / GT;             // cell slot of this thread
  const int tg = threadIdx.x % GT;
  const int q = tg >> 1, h = tg & 1;          // pencil (row / column index) and half
  const int w = threadIdx.x >> 5;             // warp
  double2* wk = reinterpret_cast<double2*>(smem + g * C::PLANE);
  int8_t (*sdelta)[kMaxN] = reinterpret_cast<int8_t (*)[kMaxN]>(smem + C::OFF_DELTA);
  double* red = reinterpret_cast<double*>(smem + C::OFF_RED) + g * C::NWG * 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  double2* tab = reinterpret_cast<double2*>(smem + C::OFF_TAB);  // [A+1][l_y][HC] (TAB_SMEM)
  load_delta(p.tp, sdelta);
  if constexpr (C::TAB_SMEM) {
    FKS_CHECK((int64_t)(p.A + 1) * n <= p.table_elems);
    const int tot = (p.A + 1) * N * C::HC;
    for (int e = threadIdx.x; e < tot; e += C::THREADS) {
      const int col = e % C::HC, ly = (e / C::HC) % N, d = e / (C::HC * N);
      tab[e] = __ldg(p.tables + (size_t)d * n + ly * N + col);
    }
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = *tmem_slot;
  // the WPQ warps w, w + 4, ... sharing a TMEM lane quarter use disjoint column ranges
  const uint32_t lane_base = tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * (C::FCOLS + C::SCOLS));
  const uint32_t taddr = lane_base;              // f^ half column (parity order)
  const uint32_t saddr = lane_base + C::FCOLS;   // f* half row (halves order)
  const int stride = gridDim.x * C::CELLS;
  // table column of this thread's pencil l_x = q: columns above N/2 read the mirror (-l_x, -l_y)
  const bool neg = q > N / 2;
  const int tcol = neg ? N - q : q;

  // cells walked CTA by CTA; a group past the end recomputes the last cell and skips its stores
  // (every lane of a warp executes the warp-collective tcgen05 instructions)
  for (int base = blockIdx.x * C::CELLS; base < p.ncells; base += stride) {
    const int itr = base + g;
    const bool active = itr < p.ncells;
    const int it = active ? itr : p.ncells - 1;
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc = cell_coord(p.tp, cell);
    {  // a3: half h of row y = q of f* (cached in TMEM), forward DIF along x -> SMEM row q (parity)
      double2 r[H];
      if (p.tp.dx == 0) {
        const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * (int64_t)n + N * q + H * h);
#pragma unroll
        for (int j = 0; j < H / 2; ++j) {
          const double2 v = __ldg(src + j);
          r[2 * j] = make_double2(v.x, 0.0);
          r[2 * j + 1] = make_double2(v.y, 0.0);
        }
      } else {
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const int x = H * h + j;
          r[j] = make_double2(gather_fstar(p.f_in, p.tp, cc, x + N * q, x, q, 0, n, sdelta), 0.0);
        }
      }
#pragma unroll
      for (int ch = 0; ch < H / 16; ++ch) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[2 * i] = __double2loint(r[ch * 16 + i].x);
          v[2 * i + 1] = __double2hiint(r[ch * 16 + i].x);
        }
        tmem_st32p(saddr + ch * 32, v);
      }
      fftp_dif<N, -1>(r, h);
#pragma unroll
      for (int m = 0; m < H; ++m) wk[swp<N>(q, 2 * m + h)] = r[m];
    }
    grp_bar(1 + g, GT);
    {  // a4: column l_x = q, rows [H h, H h + H) (halves), DIF along y -> f^ (parity) in TMEM
      double2 c[H];
#pragma unroll
      for (int j = 0; j < H; ++j) c[j] = wk[swp<N>(H * h + j, q)];
      fftp_dif<N, -1>(c, h);
#pragma unroll
      for (int ch = 0; ch < H / 8; ++ch) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[4 * i + 0] = __double2loint(c[ch * 8 + i].x);
          v[4 * i + 1] = __double2hiint(c[ch * 8 + i].x);
          v[4 * i + 2] = __double2loint(c[ch * 8 + i].y);
          v[4 * i + 3] = __double2hiint(c[ch * 8 + i].y);
        }
        tmem_st32p(taddr + ch * 32, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    double gacc[H];  // G (then Q) of row j_y = q, columns j_x in [H h, H h + H)
#pragma unroll
    for (int j = 0; j < H; ++j) gacc[j] = 0.0;
#pragma unroll 1
    for (int d = 0; d <= p.A; ++d) {
      grp_bar(1 + g, GT);  // plane free (previous row pass)
      {  // pass 0: column l_x = q, l_y = 2m + h: X = T f^, DIT IFFT along y -> SMEM column q rows [H h, +H)
        double2 c[H];
#pragma unroll
        for (int ch = 0; ch < H / 8; ++ch) {
          double2 tt[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int ly = 2 * (ch * 8 + i) + h;
            if constexpr (C::TAB_SMEM) {
              const int row = neg ? (N - ly) & (N - 1) : ly;
              tt[i] = tab[((size_t)d * N + row) * C::HC + tcol];
            } else {
              FKS_CHECK((int64_t)d * n + (int64_t)ly * N + q < p.table_elems);
              tt[i] = __ldg(p.tables + (size_t)d * n + ly * N + q);
            }
          }
          uint32_t v[32];
          tmem_ld32p(taddr + ch * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double Fx = __hiloint2double(v[4 * i + 1], v[4 * i + 0]);
            const double Fy = __hiloint2double(v[4 * i + 3], v[4 * i + 2]);
            c[ch * 8 + i] = make_double2(fma(tt[i].x, Fx, -tt[i].y * Fy), fma(tt[i].x, Fy, tt[i].y * Fx));
          }
        }
        fftp_dit<N, +1>(c, h);
#pragma unroll
        for (int j = 0; j < H; ++j) wk[swp<N>(H * h + j, q)] = c[j];
      }
      grp_bar(1 + g, GT);
      {  // pass 1: row j_y = q, inputs l_x = 2m + h from SMEM, DIT IFFT along x, accumulate
        double2 r[H];
#pragma unroll
        for (int m = 0; m < H; ++m) r[m] = wk[swp<N>(q, 2 * m + h)];
        fftp_dit<N, +1>(r, h);
        if (d < p.A) {
#pragma unroll
          for (int j = 0; j < H; ++j) gacc[j] = fma(r[j].x, r[j].y, gacc[j]);
        } else {
#pragma unroll
          for (int ch = 0; ch < H / 16; ++ch) {
            uint32_t v[32];
            tmem_ld32p(saddr + ch * 32, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const double fs = __hiloint2double(v[2 * i + 1], v[2 * i]);
              gacc[ch * 16 + i] = gacc[ch * 16 + i] - fs * r[ch * 16 + i].x;  // Q = G - f* c
            }
          }
        }
      }
    }
    double* out = p.f_out + cell * (int64_t)n + N * q + H * h;
    if (p.mode == 0) {
      if (active) {
#pragma unroll
        for (int j = 0; j < H; ++j) out[j] = gacc[j];
      }
      grp_bar(1 + g, GT);  // plane free for the next cell
      continue;
    }
    double lam[4] = {0, 0, 0, 0};
    const double vy = node_v(q, p.L, p.dv);
    if (p.project) {
      double m[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < H; ++j) {
        const double vx = node_v(H * h + j, p.L, p.dv);
        m[0] += gacc[j];
        m[1] += vx * gacc[j];
        m[2] += vy * gacc[j];
        m[3] += (vx * vx + vy * vy) * gacc[j];
      }
      // group reduction in a fixed order: lanes (shuffles), then the group's warps (SMEM)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
      }
      const int wg = tg >> 5;
      if ((tg & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) red[wg * 4 + k] = m[k];
      }
      grp_bar(1 + g, GT);
      double mu[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double s = red[k];
#pragma unroll
        for (int ww = 1; ww < C::NWG; ++ww) s += red[ww * 4 + k];
        mu[k] = s;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) s = fma(p.Ginv[a * 4 + b], mu[b], s);
        lam[a] = s;
      }
    }
    bool bad = false;
    const double* hbase = p.mode == 2 ? p.f_base + cell * (int64_t)n + N * q + H * h : nullptr;
#pragma unroll
    for (int ch = 0; ch < H / 16; ++ch) {
      uint32_t v[32];
      tmem_ld32p(saddr + ch * 32, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = ch * 16 + i;
        const double fs = __hiloint2double(v[2 * i + 1], v[2 * i]);
        const double vx = node_v(H * h + j, p.L, p.dv);
        const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * (vx * vx + vy * vy);
        double o = fma(p.dt_tau, gacc[j] - corr, fs);
        if (hbase) o = 0.5 * (o + __ldcs(hbase + j));  // Heun: (f* + E(f1)) / 2 (NEXT-4)
        bad |= !isfinite(o);
        if (active) out[j] = o;
      }
    }
    if (bad && active) atomicOr(p.nonfinite, 1);
    grp_bar(1 + g, GT);  // red / plane free for the next cell
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(512) : "memory");
}

template <int N>
static cudaError_t launchp(const StepParams& p, int nblocks, cudaStream_t s) {
  using C = CfgP<N>;
  const size_t sm = C::smem(p.A);
  if (sm > 232448) return cudaErrorInvalidValue;  // (N = 32: A <= 10 directions fit the SMEM tables)
  cudaError_t e = cudaFuncSetAttribute(k_step2dp<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_step2dp<N><<<nblocks, C::THREADS, sm, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_step2d_pair(int N, const StepParams& p, int nblocks, cudaStream_t s) {
  switch (N) {
    case 32: return launchp<32>(p, nblocks, s);
    case 64: return launchp<64>(p, nblocks, s);
    default: return cudaErrorInvalidValue;
  }
}

int cells_per_block2d_pair(int N) { return N == 32 ? CfgP<32>::CELLS : N == 64 ? CfgP<64>::CELLS : 0; }

bool step2d_pair_fits(int N, int A) {
  return (N == 32 || N == 64) && (N == 32 ? CfgP<32>::smem(A) : CfgP<64>::smem(A)) <= 232448;
}

}  // namespace fks
