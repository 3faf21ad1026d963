// HBM-bound companions of the fused step: transport-only (a1+a3), solid-cell copy and the
// moment reduction (a10).
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace fks {

// General transport (any shift size): one CTA row per cell slice, one element per thread.
__global__ void k_transport(const double* __restrict__ f_in, double* __restrict__ f_out, const TransportParams tp,
                            const uint8_t* __restrict__ solid, int64_t ncells, int n, int N, int dv) {
  __shared__ int8_t sdelta[3][kMaxN];
  load_delta(tp, sdelta);
  __syncthreads();
  for (int64_t cell = blockIdx.y; cell < ncells; cell += gridDim.y) {
    FKS_CHECK(cell < tp.ncells_total);
    const bool is_solid = solid != nullptr && solid[cell];
    const CellCoord cc = cell_coord(tp, cell);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
      const int kx = k % N, ky = (k / N) % N, kz = dv == 3 ? k / (N * N) : 0;
      const double v = is_solid ? f_in[cell * n + k] : gather_fstar(f_in, tp, cc, k, kx, ky, kz, n, sdelta);
      f_out[cell * n + k] = v;
    }
  }
}

// Transport at CFL <= 1 (every shift in {-1, 0, 1}): per cell the 3^dx possible sources are
// resolved once (source_base: neighbour cell, ghost vector or halo plane) and every element is a
// table lookup + one load; persistent CTAs walk the cells.  HBM-bound: 16 B per update.
template <int N, int DV>
__global__ void __launch_bounds__(256) k_transport_cfl1(const double* __restrict__ f_in, double* __restrict__ f_out,
                                                        const TransportParams tp, const uint8_t* __restrict__ solid,
                                                        int64_t ncells) {
  constexpr int n = DV == 3 ? N * N * N : N * N;
  __shared__ int8_t sdelta[3][kMaxN];
  __shared__ const double* sbase[27];
  __shared__ int8_t sflip[27];  // mirrored velocity components per source (specular reflection)
  load_delta(tp, sdelta);
  for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
    __syncthreads();  // sdelta loaded / the previous cell's sources no longer read
    if (threadIdx.x < 27) {
      int d[3] = {(int)threadIdx.x % 3 - 1, ((int)threadIdx.x / 3) % 3 - 1, (int)threadIdx.x / 9 - 1};
      const bool is_solid = solid != nullptr && solid[cell];
      int flip = 0;
      sbase[threadIdx.x] = is_solid ? f_in + cell * n : source_resolve(f_in, tp, cell_coord(tp, cell), d, n, flip);
      sflip[threadIdx.x] = (int8_t)flip;
    }
    __syncthreads();
    double* out = f_out + cell * n;
    // k = tid + 256 i: kx = tid % N is loop-invariant (N divides 256); all UNR loads of a batch are
    // issued before its stores (the round-1 loop relied on the compiler for that and lost ~25 % when
    // an unrelated change shifted its register allocation)
#ifndef FKS_TR_UNR
#define FKS_TR_UNR 8
#endif
    constexpr int UNR = n >= 256 * FKS_TR_UNR ? FKS_TR_UNR : (n >= 256 ? n / 256 : 1);  // whole batches
    static_assert(n < 256 || n % (256 * UNR) == 0, "whole batches");
    const int kx = threadIdx.x % N;
    const int dx0 = sdelta[0][kx] + 1;
    // few cells (C3: 400 cells for 1184 CTAs): gridDim.y CTAs share a cell, each a range of batches
    const int kspan = n / (int)gridDim.y;
    auto run = [&](auto reflect) {  // the mirror lookup only exists with specular reflection
#pragma unroll 1
      for (int k0 = (int)blockIdx.y * kspan + threadIdx.x; k0 < ((int)blockIdx.y + 1) * kspan; k0 += 256 * UNR) {
        double v[UNR];
#pragma unroll
        for (int j = 0; j < UNR; ++j) {
          const int k = k0 + 256 * j;
          const int ky = (k / N) % N, kz = DV == 3 ? k / (N * N) : 0;
          const int combo = dx0 + 3 * (sdelta[1][ky] + 1) + 9 * (sdelta[2][kz] + 1);
          int ks = k;
          if constexpr (decltype(reflect)::value)
            if (sflip[combo]) ks = mirror_k(k, kx, ky, kz, sflip[combo], N);
          FKS_CHECK(combo >= 0 && combo < 27 && ks >= 0 && ks < n && cell < tp.ncells_total);
          v[j] = __ldg(sbase[combo] + ks);
        }
#pragma unroll
        for (int j = 0; j < UNR; ++j) out[k0 + 256 * j] = v[j];
      }
    };
    if (tp.reflect) run(std::true_type{});
    else run(std::false_type{});
  }
}

cudaError_t launch_transport(const double* f_in, double* f_out, const TransportParams& tp, const uint8_t* solid,
                             int64_t ncells, int n, int N, int dv, cudaStream_t s) {
  if (ncells == 0) return cudaSuccess;
  const bool cfl1 = tp.cfl1 != 0;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned nb = (unsigned)(ncells < (int64_t)sms * 8 ? ncells : (int64_t)sms * 8);
  if (cfl1) {
    // split each cell over gridDim.y CTAs when there are fewer cells than resident CTAs (each part
    // a whole number of 2048-element batches)
    int ky = 1;
    while (n >= 2048 * 2 * ky && (int64_t)nb * ky * 2 <= (int64_t)sms * 8 && ky < 16) ky *= 2;
#define FKS_TR(NN, DD) \
  if (N == NN && dv == DD) { k_transport_cfl1<NN, DD><<<dim3(nb, ky), 256, 0, s>>>(f_in, f_out, tp, solid, ncells); return cudaGetLastError(); }
    FKS_TR(8, 2) FKS_TR(16, 2) FKS_TR(32, 2) FKS_TR(64, 2) FKS_TR(8, 3) FKS_TR(16, 3) FKS_TR(32, 3) FKS_TR(64, 3)
#undef FKS_TR
  }
  const int threads = 256;
  const int chunks = (n + threads - 1) / threads;
  dim3 grid(chunks > 64 ? 64 : chunks, (unsigned)(ncells > 65535 ? 65535 : ncells));
  k_transport<<<grid, threads, 0, s>>>(f_in, f_out, tp, solid, ncells, n, N, dv);
  return cudaGetLastError();
}

__global__ void k_copy_cells(const double* __restrict__ f_in, double* __restrict__ f_out, const int* __restrict__ cells,
                             int n) {
  const int64_t c = cells[blockIdx.x];
  const double2* src = reinterpret_cast<const double2*>(f_in + c * n);
  double2* dst = reinterpret_cast<double2*>(f_out + c * n);
  for (int k = threadIdx.x; k < n / 2; k += blockDim.x) dst[k] = src[k];
}

cudaError_t launch_copy_cells(const double* f_in, double* f_out, const int* cells, int count, int n, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_copy_cells<<<count, 256, 0, s>>>(f_in, f_out, cells, n);
  return cudaGetLastError();
}

// a2 (slab exchange): pack (or unpack) the velocity slices k_axis in sl.k of `pc` consecutive
// cells starting at first_cell: buf[p][s][r] <-> f[(first_cell + p) n + k(sl.k[s], r)], r running over
// the N^{dv-1} indices of the other velocity components in C order.  HBM-bound copy.
__global__ void k_halo_pack(double* f, int64_t first_cell, int pc, int n, int N, int dv, int axis, SliceList sl,
                            double* buf, int unpack) {
  const int m = dv == 3 ? N * N : N;
  const int64_t total = (int64_t)pc * sl.n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % m);
    const int si = (int)((e / m) % sl.n);
    const int64_t p = e / ((int64_t)m * sl.n);
    const int ks = sl.k[si];
    FKS_CHECK(si < sl.n && ks >= 0 && ks < N);
    int k;
    if (axis == 0) k = ks + N * r;                               // kx fixed: (ky[, kz]) = r
    else if (axis == 1) k = (r % N) + N * (ks + N * (r / N));     // ky fixed: kx = r % N, kz = r / N
    else k = r + N * N * ks;                                     // kz fixed: a contiguous N^2 block
    double* fp = f + (first_cell + p) * n + k;
    if (unpack) *fp = buf[e];
    else buf[e] = *fp;
  }
}

cudaError_t launch_halo_pack(const double* f, int64_t first_cell, int pc, int n, int N, int dv, int axis,
                             const SliceList& sl, double* buf, bool unpack, cudaStream_t s) {
  if (pc == 0 || sl.n == 0) return cudaSuccess;
  const int m = dv == 3 ? N * N : N;
  const int64_t total = (int64_t)pc * sl.n * m;
  const int64_t blocks = (total + 255) / 256;
  k_halo_pack<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(const_cast<double*>(f), first_cell, pc,
                                                                               n, N, dv, axis, sl, buf, unpack ? 1 : 0);
  return cudaGetLastError();
}

// a10: one CTA per cell (persistent), 16-byte loads, fixed-order reduction (warp
// shuffles, then warps in order): deterministic.  HBM-bound: 8 B read per phase-space point.
template <int N, int DV>
__global__ void __launch_bounds__(256) k_moments(const double* __restrict__ f, double* rho, double* u, double* T,
                                                 int64_t ncells, double L, double h) {
  constexpr int n = DV == 3 ? N * N * N : N * N;
  __shared__ double red[8][5];
  for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
    double m[5] = {0, 0, 0, 0, 0};
    const double2* fc = reinterpret_cast<const double2*>(f + cell * n);
#pragma unroll 4
    for (int k2 = threadIdx.x; k2 < n / 2; k2 += 256) {
      const double2 p = __ldg(fc + k2);
      const int k = 2 * k2;  // k and k + 1 share v_y, v_z (N even)
      const double vx0 = node_v(k % N, L, h), vx1 = node_v(k % N + 1, L, h), vy = node_v((k / N) % N, L, h);
      const double vz = DV == 3 ? node_v(k / (N * N), L, h) : 0.0;
      const double s = p.x + p.y;
      m[0] += s;
      m[1] += vx0 * p.x + vx1 * p.y;
      m[2] += vy * s;
      m[3] += vz * s;
      m[4] += (vx0 * vx0 + vy * vy + vz * vz) * p.x + (vx1 * vx1 + vy * vy + vz * vz) * p.y;
    }
#pragma unroll
    for (int c = 0; c < 5; ++c) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
    }
    __syncthreads();  // red free (previous cell)
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int c = 0; c < 5; ++c) red[threadIdx.x >> 5][c] = m[c];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double r0 = 0, r1 = 0, r2 = 0, r3 = 0, r4 = 0;
      for (int w = 0; w < 8; ++w) {
        r0 += red[w][0]; r1 += red[w][1]; r2 += red[w][2]; r3 += red[w][3]; r4 += red[w][4];
      }
      double cell_vol = 1.0;
      for (int a = 0; a < DV; ++a) cell_vol *= h;
      const double r = cell_vol * r0;
      const double ux = cell_vol * r1 / r, uy = cell_vol * r2 / r, uz = cell_vol * r3 / r;
      const double e = cell_vol * r4 / r;
      rho[cell] = r;
      u[cell * DV + 0] = ux;
      u[cell * DV + 1] = uy;
      if (DV == 3) u[cell * DV + 2] = uz;
      T[cell] = (e - (ux * ux + uy * uy + uz * uz)) / DV;
    }
  }
}

// Small cells (2D): one warp per cell, same arithmetic order per lane, shuffle reduction.
template <int N>
__global__ void __launch_bounds__(256) k_moments_warp(const double* __restrict__ f, double* rho, double* u, double* T,
                                                      int64_t ncells, double L, double h) {
  constexpr int n = N * N;
  const int lane = threadIdx.x & 31;
  for (int64_t cell = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); cell < ncells; cell += (int64_t)gridDim.x * 8) {
    double m[4] = {0, 0, 0, 0};
    const double2* fc = reinterpret_cast<const double2*>(f + cell * n);
#pragma unroll 4
    for (int k2 = lane; k2 < n / 2; k2 += 32) {
      const double2 p = __ldg(fc + k2);
      const int k = 2 * k2;
      const double vx0 = node_v(k % N, L, h), vx1 = node_v(k % N + 1, L, h), vy = node_v(k / N, L, h);
      const double s = p.x + p.y;
      m[0] += s;
      m[1] += vx0 * p.x + vx1 * p.y;
      m[2] += vy * s;
      m[3] += (vx0 * vx0 + vy * vy) * p.x + (vx1 * vx1 + vy * vy) * p.y;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
    }
    if (lane == 0) {
      const double cell_vol = h * h;
      const double r = cell_vol * m[0];
      const double ux = cell_vol * m[1] / r, uy = cell_vol * m[2] / r;
      const double e = cell_vol * m[3] / r;
      rho[cell] = r;
      u[cell * 2 + 0] = ux;
      u[cell * 2 + 1] = uy;
      T[cell] = (e - (ux * ux + uy * uy)) / 2;
    }
  }
}

cudaError_t launch_moments(const double* f, double* rho, double* u, double* T, int64_t ncells, int N, int dv,
                           double L, double h, cudaStream_t s) {
  if (ncells == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned nb = (unsigned)(ncells < (int64_t)sms * 8 ? ncells : (int64_t)sms * 8);
  if (dv == 2) {
    const unsigned nw = (unsigned)((ncells + 7) / 8 < (int64_t)sms * 8 ? (ncells + 7) / 8 : (int64_t)sms * 8);
    if (N == 8) { k_moments_warp<8><<<nw, 256, 0, s>>>(f, rho, u, T, ncells, L, h); return cudaGetLastError(); }
    if (N == 16) { k_moments_warp<16><<<nw, 256, 0, s>>>(f, rho, u, T, ncells, L, h); return cudaGetLastError(); }
    if (N == 32) { k_moments_warp<32><<<nw, 256, 0, s>>>(f, rho, u, T, ncells, L, h); return cudaGetLastError(); }
    if (N == 64) { k_moments_warp<64><<<nw, 256, 0, s>>>(f, rho, u, T, ncells, L, h); return cudaGetLastError(); }
  }
#define FKS_MO(NN, DD) \
  if (N == NN && dv == DD) { k_moments<NN, DD><<<nb, 256, 0, s>>>(f, rho, u, T, ncells, L, h); return cudaGetLastError(); }
  FKS_MO(4, 2) FKS_MO(8, 2) FKS_MO(16, 2) FKS_MO(32, 2) FKS_MO(4, 3) FKS_MO(8, 3) FKS_MO(16, 3) FKS_MO(32, 3) FKS_MO(64, 3)
#undef FKS_MO
  return cudaErrorInvalidValue;
}

}  // namespace fks
