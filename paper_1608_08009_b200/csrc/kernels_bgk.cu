// NEXT-2: BGK relaxation step with the conservative (projected) Maxwellian, fused with the FKS
// transport gather.  P:122-127 (eq. ibgk) Q = nu (M[f] - f); P:359-364 (eq. minimMax)
// E[U] = E~ + Phi^T (Phi Phi^T)^{-1} (Phi f - Phi E~); P:909 the 1/tau rescaling
// forward Euler; nu = rho or a constant mu; the Euler limit returns E.
//
// One CTA per cell (persistent): pass 1 gathers f* and reduces its 5 (2D: 4) moments, pass 2
// evaluates the pointwise Maxwellian and reduces its moments, pass 3 writes
// f* + (dt/tau) nu (E - f*).  f* is re-gathered (an L2 hit) instead of held: a 32^3 cell is
// 256 KiB.  Reductions are fixed-order (warp shuffles, then warps in order): deterministic.
// HBM-bound: 16 B per phase-space update (read f, write f); the Maxwellian is separable, so a
// cell needs only DV * N exponentials.
#include "common.cuh"
#include "kernels.cuh"

namespace fks {

template <int N, int DV>
__device__ __forceinline__ void phi_row(int k, double L, double h, double (&ph)[5]) {
  const double vx = node_v(k % N, L, h), vy = node_v((k / N) % N, L, h);
  const double vz = DV == 3 ? node_v(k / (N * N), L, h) : 0.0;
  ph[0] = 1.0;
  ph[1] = vx;
  ph[2] = vy;
  ph[3] = vz;
  ph[4] = vx * vx + vy * vy + vz * vz;
}

// Fixed-order block sum of m[0..4] (256 threads); every thread gets the totals.
__device__ __forceinline__ void block_sum5(double (&m)[5], double (*red)[5]) {
#pragma unroll
  for (int c = 0; c < 5; ++c) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
  }
  __syncthreads();  // red free
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int c = 0; c < 5; ++c) red[threadIdx.x >> 5][c] = m[c];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w][c];
    m[c] = s;
  }
}

template <int N, int DV>
__global__ void __launch_bounds__(256) k_bgk(const BgkParams p) {
  constexpr int n = DV == 3 ? N * N * N : N * N;
  constexpr int NM = DV + 2;  // moments: 1, v (DV), |v|^2
  __shared__ int8_t sdelta[3][kMaxN];
  __shared__ const double* sbase[27];
  __shared__ double red[8][5];
  __shared__ double sexp[3][kMaxN];  // separable Maxwellian factors exp(-(v_k - u_a)^2 / (2T))
  load_delta(p.tp, sdelta);
  const double h = p.dv;
  double vol = 1.0;
  for (int a = 0; a < DV; ++a) vol *= h;
  for (int it = blockIdx.x; it < p.ncells; it += gridDim.x) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    const CellCoord cc = cell_coord(p.tp, cell);
    __syncthreads();  // sdelta loaded / previous cell's sources no longer read
    if (p.tp.dx > 0 && p.tp.cfl1 && threadIdx.x < 27) {
      const int d[3] = {(int)threadIdx.x % 3 - 1, ((int)threadIdx.x / 3) % 3 - 1, (int)threadIdx.x / 9 - 1};
      sbase[threadIdx.x] = source_base(p.f_in, p.tp, cc, d, n);
    }
    __syncthreads();
    auto fstar = [&](int k) -> double {  // a1 + a3 for velocity k of this cell
      const int kx = k % N, ky = (k / N) % N, kz = DV == 3 ? k / (N * N) : 0;
      if (p.tp.dx == 0) return __ldg(p.f_in + cell * n + k);
      if (p.tp.cfl1) {
        const int combo = (sdelta[0][kx] + 1) + 3 * (sdelta[1][ky] + 1) + 9 * (sdelta[2][kz] + 1);
        return sbase[combo][k];
      }
      return gather_fstar(p.f_in, p.tp, cc, k, kx, ky, kz, n, sdelta);
    };
    // pass 1: moments of f*
    double m[5] = {0, 0, 0, 0, 0};
    for (int k = threadIdx.x; k < n; k += 256) {
      const double f = fstar(k);
      double ph[5];
      phi_row<N, DV>(k, p.L, h, ph);
#pragma unroll
      for (int c = 0; c < 5; ++c) m[c] = fma(ph[c], f, m[c]);
    }
    block_sum5(m, red);
    double U[5];  // Phi f* in the row order 1, v_x .. v_{DV-1}, |v|^2
    U[0] = m[0];
    for (int a = 0; a < DV; ++a) U[1 + a] = m[1 + a];
    U[DV + 1] = m[4];
    const double rho = vol * m[0];
    double u[3] = {0, 0, 0}, uu = 0.0;
    for (int a = 0; a < DV; ++a) {
      u[a] = vol * m[1 + a] / rho;
      uu += u[a] * u[a];
    }
    const double T = (vol * m[4] / rho - uu) / DV;
    const double amp = rho / pow(2.0 * 3.141592653589793 * T, 0.5 * DV);
    // the Maxwellian is a product of 1D Gaussians: DV * N exponentials per cell, not n
    if (threadIdx.x < DV * N) {
      const int a = threadIdx.x / N, k = threadIdx.x % N;
      const double w = node_v(k, p.L, h) - u[a];
      sexp[a][k] = exp(-(w * w) / (2.0 * T));
    }
    __syncthreads();
    auto maxw = [&](int k) -> double {  // pointwise Maxwellian E~
      const double e = amp * sexp[0][k % N] * sexp[1][(k / N) % N];
      return DV == 3 ? e * sexp[2][k / (N * N)] : e;
    };
    // pass 2: moments of E~, then lambda = (Phi Phi^T)^{-1} (Phi f* - Phi E~)
    double me[5] = {0, 0, 0, 0, 0};
    for (int k = threadIdx.x; k < n; k += 256) {
      const double e = maxw(k);
      double ph[5];
      phi_row<N, DV>(k, p.L, h, ph);
#pragma unroll
      for (int c = 0; c < 5; ++c) me[c] = fma(ph[c], e, me[c]);
    }
    block_sum5(me, red);
    double r[5];
    r[0] = U[0] - me[0];
    for (int a = 0; a < DV; ++a) r[1 + a] = U[1 + a] - me[1 + a];
    r[DV + 1] = U[DV + 1] - me[4];
    double lam[5] = {0, 0, 0, 0, 0};
    for (int a = 0; a < NM; ++a) {
      double s = 0.0;
      for (int b = 0; b < NM; ++b) s = fma(p.Ginv[a * NM + b], r[b], s);
      lam[a] = s;
    }
    const double nu = p.nu_rule == 0 ? rho : p.mu;
    const double c1 = p.dt_tau * nu;
    // pass 3: E = E~ + Phi^T lambda; F = f* + (dt/tau) nu (E - f*)  (or E: Euler limit)
    bool bad = false;
    double* out = p.f_out + cell * n;
    for (int k = threadIdx.x; k < n; k += 256) {
      double ph[5];
      phi_row<N, DV>(k, p.L, h, ph);
      double E = maxw(k) + lam[0];
      for (int a = 0; a < DV; ++a) E = fma(lam[1 + a], ph[1 + a], E);
      E = fma(lam[DV + 1], ph[4], E);
      const double f = fstar(k);
      const double o = p.nu_rule == 2 ? E : fma(c1, E - f, f);
      bad |= !isfinite(o);
      out[k] = o;
    }
    if (bad) atomicOr(p.nonfinite, 1);
  }
}

cudaError_t launch_bgk(int N, int dv, const BgkParams& p, int sm_count, cudaStream_t s) {
  if (p.ncells == 0) return cudaSuccess;
  const unsigned nb = (unsigned)(p.ncells < sm_count * 8 ? p.ncells : sm_count * 8);
#define FKS_BGK(NN, DD) \
  if (N == NN && dv == DD) { k_bgk<NN, DD><<<nb, 256, 0, s>>>(p); return cudaGetLastError(); }
  FKS_BGK(8, 2) FKS_BGK(16, 2) FKS_BGK(32, 2) FKS_BGK(8, 3) FKS_BGK(16, 3) FKS_BGK(32, 3)
#undef FKS_BGK
  return cudaErrorInvalidValue;
}

}  // namespace fks
