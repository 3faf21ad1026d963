// 3D fused collision / step kernel (a3-a9) for a 64^3 velocity grid.
//
// Same method as kernels3d.cu (per direction the packed complex IFFT
// z = IFFT((alpha~_p + i alpha'~_p) f^), G += Re z Im z (reading #10); the loss as the
// (A+1)-th item with table (D~, 0), Q = G - f* Re z; projection; Euler
// P:273-275 or the Heun stage), but one 64^3 complex field is 4 MiB, so a cell is owned by a group
// of P64 = 64 co-resident CTAs (launch_step3d64) and each transform goes through L2 twice:
//   CTA r owns the spectrum pencils (l_x, l_y = r, all l_z) -- f^ resident in its TMEM -- and the
//   output plane j_z = r -- the gain accumulator G in registers, f* cached in TMEM.
// Per direction: (I1) X = T f^ on the CTA's 64 pencils, IFFT along z, pencils written to the
// group's exchange buffer; group barrier; (I2) the CTA's j_z plane read back, IFFT along y
// (columns, registers -> SMEM), IFFT along x (rows, SMEM -> registers), accumulate.  The forward
// transform (a4) runs the same passes in the other order: plane FFT along x then y (F1), barrier,
// pencil FFT along z into TMEM (F2).  Two sets of exchange slots alternate (NB64 directions per
// barrier, one set each), so one barrier per batch suffices: a CTA writing batch t + 2 has passed
// barrier t + 1, which every CTA reaches only after reading batch t.  (Measured alternatives:
// profiles/r02_n64.md -- software-pipelining the next direction's pencils into the barrier wait,
// 2-4 directions per barrier, 3 CTAs per SM: all slower.)
// Every 64-point pencil is split over a lane pair (fftp.cuh): 128 threads = 64 pencils, two CTAs
// (two different groups) per SM, all CTAs co-resident (launch_step3d64).  Tables: full layout
// T[p][l_z][l_y][l_x], pre-folded as in kernels3d.cu (alpha~ = s w_p alpha_p / n,
// alpha'~ = alpha'_p / n, D~ = s D / n).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "fft.cuh"
#include "fftp.cuh"
#include "kernels.cuh"

namespace fks {

namespace {

constexpr int N64 = 64;
constexpr int H64 = 32;                  // complex values per thread of a pencil
constexpr int PL64 = N64 * N64;          // plane
constexpr int NN64 = N64 * N64 * N64;    // one cell
constexpr int P64 = 64;                  // CTAs per cell: one j_z plane / one l_y pencil plane each
constexpr int T64 = 128;                 // threads per CTA: one lane pair per pencil
#ifndef FKS_N64_CTAS
#define FKS_N64_CTAS 2
#endif
constexpr int CTAS64 = FKS_N64_CTAS;     // resident CTAs per SM (2, or 3 with f* re-gathered)
constexpr bool FS_TMEM64 = CTAS64 == 2;  // f* cached in TMEM for the loss term and the update
constexpr int TMEM64 = FS_TMEM64 ? 256 : 128;  // f^ (32 complex = 128 columns) [+ f* (32 fp64 = 64 columns)]
#ifndef FKS_N64_BATCH
#define FKS_N64_BATCH 1
#endif
constexpr int NB64 = FKS_N64_BATCH;  // directions per group barrier

// Group barrier counter and the projection partials of one group (zeroed before every launch).
struct Sync64 {
  unsigned bar;
  unsigned pad[31];
  double partial[P64][8];  // [rank][moment] of the cell in flight
};

constexpr size_t OFF_DELTA64 = (size_t)PL64 * 16;          // after the plane
constexpr size_t OFF_RED64 = OFF_DELTA64 + 3 * kMaxN;      // [4 warps][5] + lambda[5]
constexpr size_t OFF_TMEM64 = OFF_RED64 + 25 * 8;
constexpr size_t SMEM_USED64 = OFF_TMEM64 + 16;
// Requested dynamic SMEM: large enough that a third CTA never fits an SM -- its tcgen05.alloc would
// wait for columns held by the two resident CTAs of other groups while its own group waits for it.
constexpr size_t SMEM64 = CTAS64 == 2 ? 100 * 1024 : 72 * 1024;
static_assert(SMEM_USED64 <= SMEM64 && (CTAS64 + 1) * (SMEM64 + 1024) > 233472 &&
                  CTAS64 * (SMEM64 + 1024) <= 233472 && CTAS64 * TMEM64 <= 512,
              "CTAS64 CTAs per SM, never one more");

// Element (row r, column c) of the SMEM plane.  XOR swizzle on the 16-byte slots within 128 B:
// bits 1-2 from r & 3 (row sweeps: 4 rows x 2 parities per quarter warp) and bit 2 from r >> 5
// (column sweeps: rows j and 32 + j of 4 columns per quarter warp) -- conflict-free for all four
// access patterns of F1 / I2.
__device__ __forceinline__ int sw64(int r, int c) { return r * N64 + (c ^ (((r & 3) << 1) ^ ((r >> 5) << 2))); }

__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&v)[32]) {
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

__device__ __forceinline__ unsigned ld_acquire64(const unsigned* ctr) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
  return v;
}

// Barrier over the P64 CTAs of a group: the counter only grows (target = P64 x barriers so far).
// Writes before it (exchange buffer, partials) are visible to every CTA of the group after it
// (bar.sync, then thread 0's fence + release add; thread 0's acquire load, then bar.sync).
// A member that never arrives would hang the GPU: after ~2^24 polls the kernel traps instead.
__device__ __forceinline__ void group_bar(Sync64* gs, unsigned& target) {
  target += P64;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(&gs->bar) : "memory");
    unsigned spins = 0;
    while ((int)(ld_acquire64(&gs->bar) - target) < 0) {
      if (++spins == (1u << 24)) __trap();
    }
  }
  __syncthreads();
}

}  // namespace

__global__ void __launch_bounds__(T64, CTAS64) k_step3d64(const StepParams p) {
  constexpr int N = N64, H = H64, n = NN64, PL = PL64;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* pl = reinterpret_cast<double2*>(smem);  // one 64 x 64 complex plane (sw64)
  int8_t (*sdelta)[kMaxN] = reinterpret_cast<int8_t (*)[kMaxN]>(smem + OFF_DELTA64);
  double* red = reinterpret_cast<double*>(smem + OFF_RED64);  // [4][5], then lambda[5]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM64);
  const int t = threadIdx.x, q = t >> 1, h = t & 1, w = t >> 5;
  const int rank = blockIdx.x % P64, grp = blockIdx.x / P64, ngrp = gridDim.x / P64;
  Sync64* gs = reinterpret_cast<Sync64*>(p.sync) + grp;
  double2* wbuf = p.scratch + (size_t)grp * 2 * NB64 * n;  // exchange slots [j_z or l_z][l_y][l_x]
  load_delta(p.tp, sdelta);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))),
                 "n"(TMEM64)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = *tmem_slot;
  FKS_CHECK((tbase & 0xffffu) + TMEM64 <= 512u);
  const uint32_t faddr = tbase + ((uint32_t)(32 * w) << 16);  // f^ of pencil (q, rank), l_z = 2m + h
  const uint32_t saddr = faddr + 128;                          // f*(x = H h + j, y = q, z = rank)
  unsigned target = 0;  // group barriers so far x P64
  unsigned item = 0;    // exchange batches so far (slot set item & 1)

  for (int it = grp; it < p.ncells; it += ngrp) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc = cell_coord(p.tp, cell);
    // f*(x = H h + j, y = q, z = rank) when it is not cached in TMEM: gathered again (a3)
    auto fstar_at = [&](int j) -> double {
      const int x = H * h + j;
      if (p.tp.dx == 0) return __ldg(p.f_in + cell * (int64_t)n + PL * rank + N * q + x);
      return gather_fstar(p.f_in, p.tp, cc, x + N * (q + N * rank), x, q, rank, n, sdelta);
    };
    __syncthreads();  // plane / red free (previous cell)
    {  // F1 (a3 + a4): row y = q of plane z = rank: f* halves (cached in TMEM), DIF along x
      double2 r[H];
      if (p.tp.dx == 0) {
        const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * (int64_t)n + PL * rank + N * q + H * h);
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
          r[j] = make_double2(gather_fstar(p.f_in, p.tp, cc, x + N * (q + N * rank), x, q, rank, n, sdelta), 0.0);
        }
      }
      if constexpr (FS_TMEM64) {
#pragma unroll
        for (int ch = 0; ch < H / 16; ++ch) {
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            v[2 * i] = __double2loint(r[ch * 16 + i].x);
            v[2 * i + 1] = __double2hiint(r[ch * 16 + i].x);
          }
          tm_st32(saddr + ch * 32, v);
        }
      }
      fftp_dif<N, -1>(r, h);
#pragma unroll
      for (int m = 0; m < H; ++m) pl[sw64(q, 2 * m + h)] = r[m];
    }
    __syncthreads();
    {  // F1: column l_x = q, rows y halves, DIF along y -> exchange [z = rank][l_y = 2m + h][q]
      double2 c[H];
#pragma unroll
      for (int j = 0; j < H; ++j) c[j] = pl[sw64(H * h + j, q)];
      fftp_dif<N, -1>(c, h);
      double2* wb = wbuf + (size_t)((item & 1) * NB64) * n + (size_t)rank * PL + q;
#pragma unroll
      for (int m = 0; m < H; ++m) __stcg(wb + (2 * m + h) * N, c[m]);
    }
    group_bar(gs, target);
    {  // F2: pencil (l_x = q, l_y = rank), z halves, DIF along z -> f^ (l_z = 2m + h) in TMEM
      const double2* wb = wbuf + (size_t)((item & 1) * NB64) * n + (size_t)rank * N + q;
      double2 c[H];
#pragma unroll
      for (int j = 0; j < H; ++j) c[j] = __ldcg(wb + (size_t)(H * h + j) * PL);
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
        tm_st32(faddr + ch * 32, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
    ++item;
    double gacc[H];  // G (then Q) at (x = H h + j, y = q, z = rank)
#pragma unroll
    for (int j = 0; j < H; ++j) gacc[j] = 0.0;
    // the directions in batches of NB64 per group barrier (exchange slots: batch parity x NB64)
    auto pencils = [&](int d, int slot) {
        {  // I1: X = T f^ on pencil (q, rank), DIT IFFT along z -> exchange [j_z = H h + j][rank][q]
          // the next direction's table rows of this pencil plane -> L2 (read-only, one item ahead)
          if (d < p.A && t < N)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p.tables + (size_t)(d + 1) * n +
                                                                              (size_t)t * PL + (size_t)rank * N),
                         "r"((uint32_t)(N * sizeof(double2)))
                         : "memory");
          double2 c[H];
          const double2* td = p.tables + (size_t)d * n + (size_t)rank * N + q;
#pragma unroll
          for (int m = 0; m < H; ++m) {  // all 32 table loads in flight (l_z = 2m + h)
            FKS_CHECK((int64_t)d * n + (int64_t)(2 * m + h) * PL + rank * N + q < p.table_elems);
            c[m] = __ldg(td + (size_t)(2 * m + h) * PL);
          }
#pragma unroll
          for (int ch = 0; ch < H / 8; ++ch) {
            uint32_t v[32];
            tm_ld32(faddr + ch * 32, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const double Fx = __hiloint2double(v[4 * i + 1], v[4 * i + 0]);
              const double Fy = __hiloint2double(v[4 * i + 3], v[4 * i + 2]);
              const double2 tt = c[ch * 8 + i];
              c[ch * 8 + i] = make_double2(fma(tt.x, Fx, -tt.y * Fy), fma(tt.x, Fy, tt.y * Fx));
            }
          }
          fftp_dit<N, +1>(c, h);
          double2* o = wbuf + (size_t)slot * n + (size_t)rank * N + q;
#pragma unroll
          for (int j = 0; j < H; ++j) __stcg(o + (size_t)(H * h + j) * PL, c[j]);
        }
    };
    auto planes = [&](int d, int slot) {
        {  // I2: plane j_z = rank, column l_x = q, rows l_y = 2m + h, DIT IFFT along y -> SMEM
          const double2* src = wbuf + (size_t)slot * n + (size_t)rank * PL + q;
          double2 c[H];
#pragma unroll
          for (int m = 0; m < H; ++m) c[m] = __ldcg(src + (2 * m + h) * N);
          fftp_dit<N, +1>(c, h);
#pragma unroll
          for (int j = 0; j < H; ++j) pl[sw64(H * h + j, q)] = c[j];
        }
        __syncthreads();
        {  // I2: row j_y = q, columns l_x = 2m + h, DIT IFFT along x, accumulate
          double2 r[H];
#pragma unroll
          for (int m = 0; m < H; ++m) r[m] = pl[sw64(q, 2 * m + h)];
          fftp_dit<N, +1>(r, h);
          if (d < p.A) {
#pragma unroll
            for (int j = 0; j < H; ++j) gacc[j] = fma(r[j].x, r[j].y, gacc[j]);
          } else if constexpr (FS_TMEM64) {
#pragma unroll
            for (int ch = 0; ch < H / 16; ++ch) {
              uint32_t v[32];
              tm_ld32(saddr + ch * 32, v);
              asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const double fs = __hiloint2double(v[2 * i + 1], v[2 * i]);
                gacc[ch * 16 + i] = gacc[ch * 16 + i] - fs * r[ch * 16 + i].x;  // Q = G - f* c
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < H; ++j) gacc[j] = gacc[j] - fstar_at(j) * r[j].x;
          }
        }
    };
#pragma unroll 1
    for (int d0 = 0; d0 <= p.A; d0 += NB64) {
      const int nb = min(NB64, p.A + 1 - d0);
      const int slot0 = (int)(item & 1) * NB64;
#pragma unroll 1
      for (int e = 0; e < nb; ++e) pencils(d0 + e, slot0 + e);
      group_bar(gs, target);
#pragma unroll 1
      for (int e = 0; e < nb; ++e) {
        if (e > 0) __syncthreads();  // the plane of the previous direction read
        planes(d0 + e, slot0 + e);
      }
      ++item;
    }
    double* out = p.f_out + cell * (int64_t)n + PL * rank + N * q + H * h;
    if (p.mode == 0) {
#pragma unroll
      for (int j = 0; j < H; ++j) out[j] = gacc[j];
      continue;
    }
    double lam[5] = {0, 0, 0, 0, 0};
    const double vy = node_v(q, p.L, p.dv), vz = node_v(rank, p.L, p.dv);
    if (p.project) {
      double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < H; ++j) {
        const double vx = node_v(H * h + j, p.L, p.dv);
        m[0] += gacc[j];
        m[1] += vx * gacc[j];
        m[2] += vy * gacc[j];
        m[3] += vz * gacc[j];
        m[4] += (vx * vx + vy * vy + vz * vz) * gacc[j];
      }
      // fixed-order reduction: lanes, warps, then the group's ranks in order (deterministic)
#pragma unroll
      for (int k = 0; k < 5; ++k) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
      }
      if ((t & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 5; ++k) red[w * 5 + k] = m[k];
      }
      __syncthreads();
      if (t < 5) __stcg(&gs->partial[rank][t], red[t] + red[5 + t] + red[10 + t] + red[15 + t]);
      group_bar(gs, target);
      if (t == 0) {
        double mu[5] = {0, 0, 0, 0, 0};
        for (int r = 0; r < P64; ++r) {
#pragma unroll
          for (int k = 0; k < 5; ++k) mu[k] += __ldcg(&gs->partial[r][k]);
        }
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < 5; ++b) s = fma(p.Ginv[a * 5 + b], mu[b], s);
          red[20 + a] = s;
        }
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 5; ++a) lam[a] = red[20 + a];
    }
    bool bad = false;
    const double* hbase = p.mode == 2 ? p.f_base + cell * (int64_t)n + PL * rank + N * q + H * h : nullptr;
#pragma unroll
    for (int ch = 0; ch < H / 16; ++ch) {
      uint32_t v[32];
      if constexpr (FS_TMEM64) {
        tm_ld32(saddr + ch * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = ch * 16 + i;
        const double fs = FS_TMEM64 ? __hiloint2double(v[2 * i + 1], v[2 * i]) : fstar_at(j);
        const double vx = node_v(H * h + j, p.L, p.dv);
        const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * vz + lam[4] * (vx * vx + vy * vy + vz * vz);
        double o = fma(p.dt_tau, gacc[j] - corr, fs);
        if (hbase) o = 0.5 * (o + __ldcs(hbase + j));  // Heun: (f* + E(f1)) / 2 (NEXT-4)
        bad |= !isfinite(o);
        out[j] = o;
      }
    }
    if (bad) atomicOr(p.nonfinite, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(TMEM64) : "memory");
}

// The full shared-memory carveout for CTAS64 CTAs per SM.
static cudaError_t prep64() {
  cudaError_t e = cudaFuncSetAttribute(k_step3d64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM64);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_step3d64, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return e;
}

// A plain launch of at most CTAS64 CTAs per SM, all co-resident: the group barriers need every
// CTA of a group running.  Not a cooperative launch: the runtime's occupancy calculation answers
// one CTA per SM for this kernel whatever its registers / shared memory / block size (apparently
// assuming a TMEM-allocating kernel owns the SM's 512 columns), although two CTAs of 256 columns
// each run side by side (measured: 10.1 vs 15.7 ms per 128-cell step; profiles/r02_n64.md).
// max_groups3d64 counts the slots from the register file and shared memory itself; with nothing
// else on the device every CTA of the grid is resident at once, and a group barrier that is
// never completed traps after ~2^24 polls instead of hanging.
cudaError_t launch_step3d64(const StepParams& p, int ngroups, cudaStream_t s) {
  cudaError_t e = prep64();
  if (e != cudaSuccess) return e;
  k_step3d64<<<ngroups * P64, T64, SMEM64, s>>>(p);
  return cudaGetLastError();
}

int max_groups3d64() {
  if (prep64() != cudaSuccess) return 0;
  cudaFuncAttributes fa;
  int dev = 0, sms = 0, smem_sm = 0, smem_rsv = 0, regs_sm = 0;
  if (cudaFuncGetAttributes(&fa, k_step3d64) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  const int regs_cta = (fa.numRegs + 7) / 8 * 8 * T64;  // 8-register allocation granularity
  int per_sm = CTAS64;
  per_sm = std::min(per_sm, regs_sm / regs_cta);
  per_sm = std::min(per_sm, smem_sm / (int)(SMEM64 + fa.sharedSizeBytes + smem_rsv));
  if (getenv("FKS_VERBOSE"))
    fprintf(stderr, "fks: k_step3d64 %d CTAs per SM x %d SMs (%d registers, %zu B SMEM per CTA)\n", per_sm, sms,
            fa.numRegs, SMEM64);
  return per_sm * sms / P64;
}
size_t scratch_elems3d64() { return (size_t)2 * NB64 * NN64; }

size_t sync_bytes3d64() { return sizeof(Sync64); }

}  // namespace fks
