// 2D fused collision / step kernel (a3-a9) for the N = 64 velocity grid (P:1065-1075 runs 64^2).
//
// Same method as kernels2d.cu (per direction a packed complex IFFT (alpha~ + i alpha'~) f^,
// G += Re z Im z; the loss as the (A+1)-th item; projection; Euler), but a 64-point pencil does not
// fit one thread's registers next to its gain accumulator, so every pencil is split over a lane pair
// (h = lane & 1 owns 32 complex values) with one radix-2 stage across the pair through shuffles:
//   forward (DIF): thread h holds x[32h + j] (halves) -> thread h gets X[2m + h] (parity);
//   inverse (DIT): thread h holds x[2m + h] (parity) -> thread h gets X[32h + j] (halves);
// the 32-point remainders are the register FFTs of fft.cuh.  The layouts chain without reshuffles:
// forward rows (halves of f*) -> SMEM -> forward columns (halves) -> f^ in TMEM in parity order ->
// per direction the column IFFT (parity in, halves out) -> SMEM -> the row IFFT reads its parity
// inputs from SMEM and leaves thread (row q, half h) the outputs j_x in [32h, 32h + 32), which is
// exactly the f* half it cached in TMEM during the forward pass.
// A CTA of 256 threads holds 2 cells (a group of 128 threads = 64 pencil pairs per cell), one
// 64 x 64 work plane per cell in SMEM (XOR swizzle c ^ ((r & 3) << 1): conflict-free for the
// column sweeps and the strided row reads), tables from L2 (576 KiB at A = 8 do not fit SMEM).
#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace fks {

namespace {

constexpr int N64 = 64;
constexpr int THREADS64 = 256;
constexpr int GT64 = 128;                          // threads per cell
constexpr int CELLS64 = THREADS64 / GT64;          // cells per CTA
constexpr size_t PLANE64 = (size_t)N64 * N64 * 16;  // 64 KiB
constexpr int FCOLS64 = 128;                       // f^ half column: 32 complex fp64
constexpr int SCOLS64 = 64;                        // f* half row: 32 fp64
constexpr size_t OFF_DELTA64 = CELLS64 * PLANE64;
constexpr size_t OFF_RED64 = OFF_DELTA64 + 3 * kMaxN;            // [CELLS][4 warps][4] moment partials
constexpr size_t OFF_TMEM64 = (OFF_RED64 + CELLS64 * 4 * 4 * 8 + 15) / 16 * 16;
constexpr size_t SMEM64 = OFF_TMEM64 + 16;

__device__ __forceinline__ int sw64(int r, int c) { return r * N64 + (c ^ ((r & 3) << 1)); }

__device__ __forceinline__ double2 shfl_pair(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 1), __shfl_xor_sync(0xffffffffu, v.y, 1));
}

// x * exp(SIGN 2 pi i kk / 64) if `on`, else x (kk compile-time after unrolling).
template <int SIGN>
__device__ __forceinline__ double2 twiddle_if(double2 x, int kk, bool on) {
  const double2 t = twiddle<SIGN>(x, kk);
  return on ? t : x;
}

// DIF: a[j] = x[32h + j] -> a[m] = X[2m + h]  (X_k = sum_j x_j exp(SIGN 2 pi i j k / 64))
template <int SIGN>
__device__ __forceinline__ void fft64_dif_pair(double2 (&a)[32], int h) {
  const double sg = h ? -1.0 : 1.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double2 b = shfl_pair(a[j]);
    // h = 0: x_j + x_{j+32};  h = 1: (x_j - x_{j+32}) W^j  (b is the partner's value)
    const double2 u = make_double2(b.x + sg * a[j].x, b.y + sg * a[j].y);
    a[j] = twiddle_if<SIGN>(u, j, h != 0);
  }
  fft<32, SIGN>(a);
}

// DIT: a[m] = x[2m + h] -> a[j] = X[32h + j]
template <int SIGN>
__device__ __forceinline__ void fft64_dit_pair(double2 (&a)[32], int h) {
  fft<32, SIGN>(a);  // h = 0: E_k (even inputs), h = 1: O_k (odd inputs)
  const double sg = h ? -1.0 : 1.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double2 t = twiddle_if<SIGN>(a[k], k, h != 0);  // h = 1: W^k O_k
    const double2 b = shfl_pair(t);
    // h = 0: X_k = E_k + W^k O_k;  h = 1: X_{k+32} = E_k - W^k O_k
    a[k] = make_double2(b.x + sg * t.x, b.y + sg * t.y);
  }
}

__device__ __forceinline__ void tmem_st32_64(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld32_64(uint32_t taddr, uint32_t (&v)[32]) {
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

}  // namespace

__global__ void __launch_bounds__(THREADS64, 1) k_step2d64(const StepParams p) {
  constexpr int N = N64, n = N64 * N64;
  extern __shared__ __align__(128) unsigned char smem[];
  const int g = threadIdx.x / GT64;           // cell slot of this thread
  const int tg = threadIdx.x % GT64;
  const int q = tg >> 1, h = tg & 1;          // pencil (row / column index) and half
  const int w = threadIdx.x >> 5;             // warp
  double2* wk = reinterpret_cast<double2*>(smem + g * PLANE64);
  int8_t (*sdelta)[kMaxN] = reinterpret_cast<int8_t (*)[kMaxN]>(smem + OFF_DELTA64);
  double* red = reinterpret_cast<double*>(smem + OFF_RED64) + g * 16;  // [4 warps][4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM64);
  load_delta(p.tp, sdelta);
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
  // warps w and w + 4 share a TMEM lane quarter: disjoint column ranges [0, 192) and [192, 384)
  const uint32_t lane_base = tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * (FCOLS64 + SCOLS64));
  const uint32_t taddr = lane_base;              // f^ half column (parity order)
  const uint32_t saddr = lane_base + FCOLS64;    // f* half row (halves order)
  const int stride = gridDim.x * CELLS64;

  // cells walked CTA by CTA; a group past the end recomputes the last cell and skips its stores
  // (every lane of a warp executes the warp-collective tcgen05 instructions)
  for (int base = blockIdx.x * CELLS64; base < p.ncells; base += stride) {
    const int itr = base + g;
    const bool active = itr < p.ncells;
    const int it = active ? itr : p.ncells - 1;
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc = cell_coord(p.tp, cell);
    {  // a3: half h of row y = q of f* (cached in TMEM), forward DIF along x -> SMEM row q (parity)
      double2 r[32];
      if (p.tp.dx == 0) {
        const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * (int64_t)n + N * q + 32 * h);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double2 v = __ldg(src + j);
          r[2 * j] = make_double2(v.x, 0.0);
          r[2 * j + 1] = make_double2(v.y, 0.0);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int x = 32 * h + j;
          r[j] = make_double2(gather_fstar(p.f_in, p.tp, cc, x + N * q, x, q, 0, n, sdelta), 0.0);
        }
      }
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[2 * i] = __double2loint(r[ch * 16 + i].x);
          v[2 * i + 1] = __double2hiint(r[ch * 16 + i].x);
        }
        tmem_st32_64(saddr + ch * 32, v);
      }
      fft64_dif_pair<-1>(r, h);
#pragma unroll
      for (int m = 0; m < 32; ++m) wk[sw64(q, 2 * m + h)] = r[m];
    }
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT64) : "memory");
    {  // a4: column l_x = q, rows [32h, 32h + 32) (halves), DIF along y -> f^ (parity) in TMEM
      double2 c[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) c[j] = wk[sw64(32 * h + j, q)];
      fft64_dif_pair<-1>(c, h);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[4 * i + 0] = __double2loint(c[ch * 8 + i].x);
          v[4 * i + 1] = __double2hiint(c[ch * 8 + i].x);
          v[4 * i + 2] = __double2loint(c[ch * 8 + i].y);
          v[4 * i + 3] = __double2hiint(c[ch * 8 + i].y);
        }
        tmem_st32_64(taddr + ch * 32, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    double gacc[32];  // G (then Q) of row j_y = q, columns j_x in [32h, 32h + 32)
#pragma unroll
    for (int j = 0; j < 32; ++j) gacc[j] = 0.0;
#pragma unroll 1
    for (int d = 0; d <= p.A; ++d) {
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT64) : "memory");  // plane free (previous row pass)
      {  // pass 0: column l_x = q, l_y = 2m + h: X = T f^, DIT IFFT along y -> SMEM column q rows [32h, +32)
        double2 c[32];
        const double2* T = p.tables + (size_t)d * n + q;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          double2 tt[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int ly = 2 * (ch * 8 + i) + h;
            FKS_CHECK((int64_t)d * n + (int64_t)ly * N + q < p.table_elems);
            tt[i] = __ldg(T + ly * N);
          }
          uint32_t v[32];
          tmem_ld32_64(taddr + ch * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double Fx = __hiloint2double(v[4 * i + 1], v[4 * i + 0]);
            const double Fy = __hiloint2double(v[4 * i + 3], v[4 * i + 2]);
            c[ch * 8 + i] = make_double2(fma(tt[i].x, Fx, -tt[i].y * Fy), fma(tt[i].x, Fy, tt[i].y * Fx));
          }
        }
        fft64_dit_pair<+1>(c, h);
#pragma unroll
        for (int j = 0; j < 32; ++j) wk[sw64(32 * h + j, q)] = c[j];
      }
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT64) : "memory");
      {  // pass 1: row j_y = q, inputs l_x = 2m + h from SMEM, DIT IFFT along x, accumulate
        double2 r[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) r[m] = wk[sw64(q, 2 * m + h)];
        fft64_dit_pair<+1>(r, h);
        if (d < p.A) {
#pragma unroll
          for (int j = 0; j < 32; ++j) gacc[j] = fma(r[j].x, r[j].y, gacc[j]);
        } else {
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            uint32_t v[32];
            tmem_ld32_64(saddr + ch * 32, v);
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
    double* out = p.f_out + cell * (int64_t)n + N * q + 32 * h;
    if (p.mode == 0) {
      if (active) {
#pragma unroll
        for (int j = 0; j < 32; ++j) out[j] = gacc[j];
      }
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT64) : "memory");  // plane free for the next cell
      continue;
    }
    double lam[4] = {0, 0, 0, 0};
    const double vy = node_v(q, p.L, p.dv);
    if (p.project) {
      double m[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double vx = node_v(32 * h + j, p.L, p.dv);
        m[0] += gacc[j];
        m[1] += vx * gacc[j];
        m[2] += vy * gacc[j];
        m[3] += (vx * vx + vy * vy) * gacc[j];
      }
      // group reduction in a fixed order: lanes (shuffles), then the group's 4 warps (SMEM)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
      }
      const int wg = (tg >> 5);
      if ((tg & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) red[wg * 4 + k] = m[k];
      }
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT64) : "memory");
      double mu[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) mu[k] = ((red[k] + red[4 + k]) + red[8 + k]) + red[12 + k];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) s = fma(p.Ginv[a * 4 + b], mu[b], s);
        lam[a] = s;
      }
    }
    bool bad = false;
    const double* hbase = p.mode == 2 ? p.f_base + cell * (int64_t)n + N * q + 32 * h : nullptr;
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
      uint32_t v[32];
      tmem_ld32_64(saddr + ch * 32, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = ch * 16 + i;
        const double fs = __hiloint2double(v[2 * i + 1], v[2 * i]);
        const double vx = node_v(32 * h + j, p.L, p.dv);
        const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * (vx * vx + vy * vy);
        double o = fma(p.dt_tau, gacc[j] - corr, fs);
        if (hbase) o = 0.5 * (o + __ldcs(hbase + j));  // Heun: (f* + E(f1)) / 2 (NEXT-4)
        bad |= !isfinite(o);
        if (active) out[j] = o;
      }
    }
    if (bad && active) atomicOr(p.nonfinite, 1);
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT64) : "memory");  // red / plane free for the next cell
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(512) : "memory");
}

cudaError_t launch_step2d64(const StepParams& p, int nblocks, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_step2d64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM64);
  if (e != cudaSuccess) return e;
  k_step2d64<<<nblocks, THREADS64, SMEM64, s>>>(p);
  return cudaGetLastError();
}

int cells_per_block2d64() { return CELLS64; }

}  // namespace fks
