// Fused collision / step kernel (a3-a9) for the smallest velocity grids, N = 4 (2D: n = 16,
// 3D: n = 64 points per cell).
//
// Same method as the other step kernels (per direction z = IDFT((alpha~ + i alpha'~) f^),
// G += Re z Im z, reading #10; the loss as the (A+1)-th item, Q = G - f* Re z;
// projection; Euler P:273-275 or the Heun stage), on a cell too small for the pencil-
// per-thread designs: one thread per velocity point, the cell's transforms done in shared memory as
// dv passes of 4-point DFTs (the radix-4 butterfly; exact twiddles 1, +-i, -1).  CELLS cells per
// 256-thread CTA, persistent over cells.  Tables in the full layout T[p][k] (fks_api.cu).
// Nothing here is bandwidth- or FLOP-bound at these sizes: the kernel exists so that the N range of
// the boundary (4 <= N <= 64) is covered by the same fused path.
#include "common.cuh"
#include "kernels.cuh"

namespace fks {

namespace {

template <int N, int DV>
struct CfgS {
  static constexpr int n = DV == 3 ? N * N * N : N * N;
  static constexpr int THREADS = 256;
  static constexpr int CELLS = THREADS / n;
  static_assert(THREADS % n == 0, "whole cells per CTA");
};

// One pass of N-point DFTs along axis a over the cell's n points, thread k writing point k:
// out[k] = sum_m in[k with index_a = m] exp(SIGN 2 pi i idx_a(k) m / N).
template <int N, int DV, int SIGN>
__device__ __forceinline__ double2 dft_axis(const double2* in, int k, int a) {
  constexpr int st[3] = {1, N, N * N};
  const int s = st[a];
  const int ia = (k / s) % N;
  const double2* base = in + (k - ia * s);
  double re = 0.0, im = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) {
    const int e = (ia * m) % N;  // exp(SIGN 2 pi i e / N), N = 4: 1, SIGN i, -1, -SIGN i
    const double2 v = base[m * s];
    if (e == 0) { re += v.x; im += v.y; }
    else if (e == N / 2) { re -= v.x; im -= v.y; }
    else if ((e == N / 4) == (SIGN > 0)) { re -= v.y; im += v.x; }  // * i
    else { re += v.y; im -= v.x; }                                     // * (-i)
  }
  return make_double2(re, im);
}

}  // namespace

template <int N, int DV>
__global__ void __launch_bounds__(256) k_step_small(const StepParams p) {
  using C = CfgS<N, DV>;
  constexpr int n = C::n;
  static_assert(N == 4, "the +-i twiddle cases above are the 4-point DFT");
  __shared__ int8_t sdelta[3][kMaxN];
  __shared__ double2 buf[2][C::CELLS][n];
  __shared__ double2 fh[C::CELLS][n];
  __shared__ double red[C::CELLS][5];
  load_delta(p.tp, sdelta);
  const int g = threadIdx.x / n, k = threadIdx.x % n;
  const int kx = k % N, ky = (k / N) % N, kz = DV == 3 ? k / (N * N) : 0;
  const double vx = node_v(kx, p.L, p.dv), vy = node_v(ky, p.L, p.dv), vz = DV == 3 ? node_v(kz, p.L, p.dv) : 0.0;
  const double v2 = vx * vx + vy * vy + vz * vz;
  for (int base = blockIdx.x * C::CELLS; base < p.ncells; base += gridDim.x * C::CELLS) {
    const int itr = base + g;
    const bool active = itr < p.ncells;
    const int it = active ? itr : p.ncells - 1;  // past the end: recompute the last cell, no stores
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    __syncthreads();  // sdelta loaded / the previous cell's buffers free
    const CellCoord cc = cell_coord(p.tp, cell);
    const double fs = gather_fstar(p.f_in, p.tp, cc, k, kx, ky, kz, n, sdelta);  // a3
    // a4: forward transform (unnormalised; 1/n is folded into the tables)
    buf[0][g][k] = make_double2(fs, 0.0);
    int cur = 0;
#pragma unroll
    for (int a = 0; a < DV; ++a) {
      __syncthreads();
      buf[cur ^ 1][g][k] = dft_axis<N, DV, -1>(buf[cur][g], k, a);
      cur ^= 1;
    }
    __syncthreads();
    fh[g][k] = buf[cur][g][k];
    double gacc = 0.0;
    for (int d = 0; d <= p.A; ++d) {
      FKS_CHECK((int64_t)d * n + k < p.table_elems);
      const double2 t = p.tables[(size_t)d * n + k];
      const double2 F = fh[g][k];
      __syncthreads();  // every thread's previous reads of buf done
      buf[0][g][k] = make_double2(fma(t.x, F.x, -t.y * F.y), fma(t.x, F.y, t.y * F.x));
      cur = 0;
#pragma unroll
      for (int a = 0; a < DV; ++a) {
        __syncthreads();
        buf[cur ^ 1][g][k] = dft_axis<N, DV, +1>(buf[cur][g], k, a);
        cur ^= 1;
      }
      __syncthreads();
      const double2 z = buf[cur][g][k];
      if (d < p.A) gacc = fma(z.x, z.y, gacc);
      else gacc = gacc - fs * z.x;  // Q = G - f* c
    }
    double* out = p.f_out + cell * (int64_t)n + k;
    if (p.mode == 0) {
      if (active) *out = gacc;
      continue;
    }
    double lam[5] = {0, 0, 0, 0, 0};
    if (p.project) {
      // the cell's n threads reduce its 5 moments in a fixed order (thread 0 of the cell, serial)
      __syncthreads();
      buf[0][g][k] = make_double2(gacc, 0.0);
      __syncthreads();
      if (k == 0) {
        double m[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < n; ++j) {
          const double q = buf[0][g][j].x;
          const double ux = node_v(j % N, p.L, p.dv), uy = node_v((j / N) % N, p.L, p.dv);
          const double uz = DV == 3 ? node_v(j / (N * N), p.L, p.dv) : 0.0;
          m[0] += q;
          m[1] += ux * q;
          m[2] += uy * q;
          m[3] += uz * q;
          m[4] += (ux * ux + uy * uy + uz * uz) * q;
        }
        double mu[5];  // Phi row order 1, v_0 .. v_{DV-1}, |v|^2 (Ginv is (DV+2)^2)
        constexpr int M = DV + 2;
        mu[0] = m[0];
        for (int a = 0; a < DV; ++a) mu[1 + a] = m[1 + a];
        mu[M - 1] = m[4];
        for (int a = 0; a < M; ++a) {
          double s = 0.0;
          for (int b = 0; b < M; ++b) s = fma(p.Ginv[a * M + b], mu[b], s);
          red[g][a] = s;
        }
      }
      __syncthreads();
      constexpr int M = DV + 2;
      lam[0] = red[g][0];
      lam[1] = red[g][1];
      lam[2] = red[g][2];
      if (DV == 3) lam[3] = red[g][3];
      lam[4] = red[g][M - 1];
    }
    const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * vz + lam[4] * v2;
    double o = fma(p.dt_tau, gacc - corr, fs);
    if (p.mode == 2) o = 0.5 * (o + p.f_base[cell * (int64_t)n + k]);  // Heun: (f* + E(f1)) / 2 (NEXT-4)
    if (!isfinite(o) && active) atomicOr(p.nonfinite, 1);
    if (active) *out = o;
  }
}

cudaError_t launch_step_small(int N, int dv, const StepParams& p, int sm_count, cudaStream_t s) {
  if (N != 4) return cudaErrorInvalidValue;
  const int cells = dv == 3 ? CfgS<4, 3>::CELLS : CfgS<4, 2>::CELLS;
  const int64_t need = (p.ncells + cells - 1) / cells;
  const unsigned nb = (unsigned)(need < (int64_t)sm_count * 8 ? need : (int64_t)sm_count * 8);
  if (dv == 3) k_step_small<4, 3><<<nb, 256, 0, s>>>(p);
  else k_step_small<4, 2><<<nb, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace fks
