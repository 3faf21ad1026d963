// HBM-bound companions of the fused step: transport-only (a1+a3), solid-cell copy and the
// moment reduction (a10).
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
  load_delta(tp, sdelta);
  for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
    __syncthreads();  // sdelta loaded / the previous cell's sources no longer read
    if (threadIdx.x < 27) {
      const int d[3] = {(int)threadIdx.x % 3 - 1, ((int)threadIdx.x / 3) % 3 - 1, (int)threadIdx.x / 9 - 1};
      const bool is_solid = solid != nullptr && solid[cell];
      sbase[threadIdx.x] = is_solid ? f_in + cell * n : source_base(f_in, tp, cell_coord(tp, cell), d, n);
    }
    __syncthreads();
    double* out = f_out + cell * n;
#pragma unroll 8
    for (int k = threadIdx.x; k < n; k += 256) {
      const int kx = k % N, ky = (k / N) % N, kz = DV == 3 ? k / (N * N) : 0;
      const int combo = (sdelta[0][kx] + 1) + 3 * (sdelta[1][ky] + 1) + 9 * (sdelta[2][kz] + 1);
      out[k] = __ldg(sbase[combo] + k);
    }
  }
}

cudaError_t launch_transport(const double* f_in, double* f_out, const TransportParams& tp, const uint8_t* solid,
                             int64_t ncells, int n, int N, int dv, cudaStream_t s) {
  if (ncells == 0) return cudaSuccess;
  bool cfl1 = true;  // rows a >= dx are zero
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < N; ++k) cfl1 &= tp.delta[a][k] >= -1 && tp.delta[a][k] <= 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned nb = (unsigned)(ncells < (int64_t)sms * 8 ? ncells : (int64_t)sms * 8);
  if (cfl1) {
#define FKS_TR(NN, DD) \
  if (N == NN && dv == DD) { k_transport_cfl1<NN, DD><<<nb, 256, 0, s>>>(f_in, f_out, tp, solid, ncells); return cudaGetLastError(); }
    FKS_TR(8, 2) FKS_TR(16, 2) FKS_TR(32, 2) FKS_TR(8, 3) FKS_TR(16, 3) FKS_TR(32, 3)
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

// a10: one CTA per cell, fixed-order tree reduction (deterministic).
__global__ void k_moments(const double* __restrict__ f, double* rho, double* u, double* T, int N, int dv, double L,
                          double h) {
  __shared__ double red[5][256];
  const int64_t cell = blockIdx.x;
  const int n = dv == 3 ? N * N * N : N * N;
  double m[5] = {0, 0, 0, 0, 0};
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double fk = f[cell * n + k];
    const double vx = node_v(k % N, L, h), vy = node_v((k / N) % N, L, h);
    const double vz = dv == 3 ? node_v(k / (N * N), L, h) : 0.0;
    m[0] += fk;
    m[1] += vx * fk;
    m[2] += vy * fk;
    m[3] += vz * fk;
    m[4] += (vx * vx + vy * vy + vz * vz) * fk;
  }
  for (int c = 0; c < 5; ++c) red[c][threadIdx.x] = m[c];
  __syncthreads();
  for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int c = 0; c < 5; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double cell_vol = 1.0;
    for (int a = 0; a < dv; ++a) cell_vol *= h;
    const double r = cell_vol * red[0][0];
    const double ux = cell_vol * red[1][0] / r, uy = cell_vol * red[2][0] / r, uz = cell_vol * red[3][0] / r;
    const double e = cell_vol * red[4][0] / r;
    rho[cell] = r;
    u[cell * dv + 0] = ux;
    u[cell * dv + 1] = uy;
    if (dv == 3) u[cell * dv + 2] = uz;
    T[cell] = (e - (ux * ux + uy * uy + uz * uz)) / dv;
  }
}

cudaError_t launch_moments(const double* f, double* rho, double* u, double* T, int64_t ncells, int N, int dv,
                           double L, double h, cudaStream_t s) {
  if (ncells == 0) return cudaSuccess;
  k_moments<<<(unsigned)ncells, 256, 0, s>>>(f, rho, u, T, N, dv, L, h);
  return cudaGetLastError();
}

}  // namespace fks
