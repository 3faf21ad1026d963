// NEXT-2: BGK relaxation step with the conservative (projected) Maxwellian, fused with the FKS
// transport gather.  P:122-127 (eq. ibgk) Q = nu (M[f] - f); P:359-364 (eq. minimMax)
// E[U] = E~ + Phi^T (Phi Phi^T)^{-1} (Phi f - Phi E~); P:909 the 1/tau rescaling
// forward Euler; nu = rho or a constant mu; the Euler limit returns E.
//
// One CTA per cell (persistent): pass 1 gathers f* and reduces its 5 (2D: 4) moments, the
// Maxwellian's moments come from 1D sums (it is separable, O(DV N) work), pass 3 writes
// f* + (dt/tau) nu (E - f*).  f* is re-gathered (an L2 hit) instead of held: a 32^3 cell is
// 256 KiB.  Reductions are fixed-order (warp shuffles, then warps in order): deterministic.
// HBM-bound: 16 B per phase-space update (read f, write f); the Maxwellian is separable, so a
// cell needs only DV * N exponentials.
#include <cstdlib>

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

// Fixed-order block sum of m[0..4] (NT threads); every thread gets the totals.
template <int NT>
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
    for (int w = 0; w < NT / 32; ++w) s += red[w][c];
    m[c] = s;
  }
}

// NT threads per CTA.  The CTA count is chosen so that the cells in flight (one per CTA, plus the
// prefetched next one) stay L2-resident between pass 1 and pass 3 (see launch_bgk).
template <int N, int DV, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bgk(const BgkParams p, const int prefetch) {
  constexpr int n = DV == 3 ? N * N * N : N * N;
  constexpr int NM = DV + 2;  // moments: 1, v (DV), |v|^2
  __shared__ int8_t sdelta[3][kMaxN];
  __shared__ const double* sbase[27];
  __shared__ int8_t sflip[27];
  __shared__ double red[NT / 32][5];
  __shared__ double sexp[3][kMaxN];  // separable Maxwellian factors exp(-(v_k - u_a)^2 / (2T))
  load_delta(p.tp, sdelta);
  const double h = p.dv;
  double vol = 1.0;
  for (int a = 0; a < DV; ++a) vol *= h;
  for (int it = blockIdx.x; it < p.ncells; it += gridDim.x) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc = cell_coord(p.tp, cell);
    __syncthreads();  // sdelta loaded / previous cell's sources no longer read
    if (p.tp.dx > 0 && p.tp.cfl1 && threadIdx.x < 27) {
      int d[3] = {(int)threadIdx.x % 3 - 1, ((int)threadIdx.x / 3) % 3 - 1, (int)threadIdx.x / 9 - 1};
      int flip = 0;
      sbase[threadIdx.x] = source_resolve(p.f_in, p.tp, cc, d, n, flip);
      sflip[threadIdx.x] = (int8_t)flip;
    }
    __syncthreads();
    auto fstar = [&](int k) -> double {  // a1 + a3 for velocity k of this cell
      const int kx = k % N, ky = (k / N) % N, kz = DV == 3 ? k / (N * N) : 0;
      if (p.tp.dx == 0) return __ldg(p.f_in + cell * n + k);
      if (p.tp.cfl1) {
        const int combo = (sdelta[0][kx] + 1) + 3 * (sdelta[1][ky] + 1) + 9 * (sdelta[2][kz] + 1);
        return sbase[combo][sflip[combo] ? mirror_k(k, kx, ky, kz, sflip[combo], N) : k];
      }
      return gather_fstar(p.f_in, p.tp, cc, k, kx, ky, kz, n, sdelta);
    };
    // the next cell of this CTA (homogeneous case: contiguous) -> L2 while this one is processed
    if (prefetch && p.tp.dx == 0 && threadIdx.x == 0 && !p.cell_list && it + gridDim.x < p.ncells)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p.f_in + (int64_t)(it + gridDim.x) * n),
                   "r"((uint32_t)(n * sizeof(double)))
                   : "memory");
    // pass 1: moments of f* (homogeneous cells: 16-byte loads, two velocities per thread)
    double m[5] = {0, 0, 0, 0, 0};
    if (p.tp.dx == 0) {
      const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * n);
#pragma unroll 4
      for (int k2 = threadIdx.x; k2 < n / 2; k2 += NT) {
        const double2 f2 = __ldg(src + k2);
        double ph[5], pq[5];
        phi_row<N, DV>(2 * k2, p.L, h, ph);
        phi_row<N, DV>(2 * k2 + 1, p.L, h, pq);
#pragma unroll
        for (int c = 0; c < 5; ++c) m[c] = fma(pq[c], f2.y, fma(ph[c], f2.x, m[c]));
      }
    } else {
#pragma unroll 4
      for (int k = threadIdx.x; k < n; k += NT) {
        const double f = fstar(k);
        double ph[5];
        phi_row<N, DV>(k, p.L, h, ph);
#pragma unroll
        for (int c = 0; c < 5; ++c) m[c] = fma(ph[c], f, m[c]);
      }
    }
    block_sum5<NT>(m, red);
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
    // pass 2: moments of E~, then lambda = (Phi Phi^T)^{-1} (Phi f* - Phi E~).  E~ and every row of
    // Phi are separable on the tensor velocity grid, so Sum_k E~(k) Phi(k) is a product of 1D sums
    // S0_a = Sum e_a, S1_a = Sum v e_a, S2_a = Sum v^2 e_a (the same finite sum, reordered).
    double S0[3] = {1, 1, 1}, S1[3] = {0, 0, 0}, S2[3] = {0, 0, 0};
    for (int a = 0; a < DV; ++a) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int k = 0; k < N; ++k) {
        const double e = sexp[a][k], v = node_v(k, p.L, h);
        s0 += e;
        s1 = fma(v, e, s1);
        s2 = fma(v * v, e, s2);
      }
      S0[a] = s0;
      S1[a] = s1;
      S2[a] = s2;
    }
    double me[5];
    me[0] = amp * S0[0] * S0[1] * S0[2];
    me[1] = amp * S1[0] * S0[1] * S0[2];
    me[2] = amp * S0[0] * S1[1] * S0[2];
    me[3] = amp * S0[0] * S0[1] * S1[2];
    me[4] = amp * (S2[0] * S0[1] * S0[2] + S0[0] * S2[1] * S0[2] + (DV == 3 ? S0[0] * S0[1] * S2[2] : 0.0));
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
    auto update = [&](int k, double f) {
      double ph[5];
      phi_row<N, DV>(k, p.L, h, ph);
      double E = maxw(k) + lam[0];
      for (int a = 0; a < DV; ++a) E = fma(lam[1 + a], ph[1 + a], E);
      E = fma(lam[DV + 1], ph[4], E);
      const double o = p.nu_rule == 2 ? E : fma(c1, E - f, f);
      bad |= !isfinite(o);
      return o;
    };
    if (p.tp.dx == 0) {
      const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * n);
      double2* dst = reinterpret_cast<double2*>(out);
#pragma unroll 4
      for (int k2 = threadIdx.x; k2 < n / 2; k2 += NT) {
        const double2 f2 = __ldg(src + k2);
        const double o0 = update(2 * k2, f2.x), o1 = update(2 * k2 + 1, f2.y);
        dst[k2] = make_double2(o0, o1);
      }
    } else {
      // with transport, pass 3 walks the cell backwards: the neighbour lines pass 1 gathered last
      // are the likeliest L2 hits (C4 shape, measured without the solid mask: 3.43 -> 3.21 ms;
      // homogeneous cells: slower, forward)
#pragma unroll 4
      for (int k = n - 1 - threadIdx.x; k >= 0; k -= NT) out[k] = update(k, fstar(k));
    }
    if (bad) atomicOr(p.nonfinite, 1);
  }
}

// 3D N = 32 with f* held in tensor memory between the passes (round-2 fix of the pass-3 re-read):
// one CTA of 512 threads per SM owns all 512 TMEM columns x 128 lanes = 256 KiB = one 32^3 fp64
// cell.  Thread t handles k = t + 512 j (j < 64; coalesced 256-byte warp accesses): pass 1 gathers
// f* in batches of 16 (all loads in flight), accumulates the moments and parks the batch in its
// TMEM lane (warps w and w + 4, w + 8, w + 12 share a lane quarter: column block w >> 2); pass 3
// reads f* back from TMEM instead of re-gathering it -- one HBM read and one write per update.
// Same arithmetic as k_bgk.
__device__ __forceinline__ void tm_st16(uint32_t taddr, const double (&f)[16]) {
  uint32_t v[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[2 * i] = __double2loint(f[i]);
    v[2 * i + 1] = __double2hiint(f[i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tm_ld16(uint32_t taddr, double (&f)[16]) {
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __hiloint2double(v[2 * i + 1], v[2 * i]);
}

template <int BW>  // gathers in flight per thread in pass 1 (16 or 32)
__global__ void __launch_bounds__(512, 1) k_bgk_tmem32(const BgkParams p) {
  constexpr int N = 32, DV = 3, NT = 512, n = N * N * N, NM = 5;
  constexpr int NB = n / NT / 16;  // TMEM chunks of 16 doubles per thread (4)
  constexpr int CPB = BW / 16;     // chunks per gather batch
  __shared__ int8_t sdelta[3][kMaxN];
  __shared__ const double* sbase[27];
  __shared__ int8_t sflip[27];
  __shared__ double red[NT / 32][5];
  __shared__ double sexp[3][kMaxN];
  __shared__ uint32_t tmem_slot;
  load_delta(p.tp, sdelta);
  const int t = threadIdx.x, w = t >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_slot))),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t taddr = tmem_slot + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * (NB * 32));
  const double h = p.dv;
  const double vol = h * h * h;
  // k = t + 512 j: kx = t % 32 is fixed per thread, ky takes two values (ky0 for even j, ky0 + 16
  // for odd j), kz = j >> 1: the moment sums and the Maxwellian factor by parity (per-thread
  // constants for x and y), only the z parts vary per element.
  const int kx = t % N, ky0 = t / N;
  const double vx = node_v(kx, p.L, h);
  const double vy[2] = {node_v(ky0, p.L, h), node_v(ky0 + 16, p.L, h)};
  for (int it = blockIdx.x; it < p.ncells; it += gridDim.x) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc = cell_coord(p.tp, cell);
    __syncthreads();  // sdelta loaded / previous cell's sources, red and sexp no longer read
    if (p.tp.dx > 0 && p.tp.cfl1 && t < 27) {
      int d[3] = {t % 3 - 1, (t / 3) % 3 - 1, t / 9 - 1};
      int flip = 0;
      sbase[t] = source_resolve(p.f_in, p.tp, cc, d, n, flip);
      sflip[t] = (int8_t)flip;
    }
    __syncthreads();
    // combo = cxy[parity] + 9 (delta_z + 1): the x and y shifts are per-thread constants
    const int cxy[2] = {(sdelta[0][kx] + 1) + 3 * (sdelta[1][ky0] + 1), (sdelta[0][kx] + 1) + 3 * (sdelta[1][ky0 + 16] + 1)};
    double s0[2] = {0, 0};    // sum f* per ky parity
    double sz = 0.0, szz = 0.0;  // sum v_z f*, sum v_z^2 f*
#pragma unroll 1
    for (int bb = 0; bb < NB; bb += CPB) {  // pass 1: BW gathers in flight, moments, park in TMEM
      double f[BW];
#pragma unroll
      for (int i = 0; i < BW; ++i) {
        const int j = 16 * bb + i;
        const int k = t + NT * j, ky = ky0 + 16 * (i & 1), kz = j >> 1;
        if (p.tp.dx == 0) {
          f[i] = __ldg(p.f_in + cell * n + k);
        } else if (p.tp.cfl1) {
          const int combo = cxy[i & 1] + 9 * (sdelta[2][kz] + 1);
          const int fl = sflip[combo];
          f[i] = __ldg(sbase[combo] + (fl ? mirror_k(k, kx, ky, kz, fl, N) : k));
        } else {
          f[i] = gather_fstar(p.f_in, p.tp, cc, k, kx, ky, kz, n, sdelta);
        }
      }
#pragma unroll
      for (int i = 0; i < BW; ++i) {
        const int j = 16 * bb + i;
        const double vz = node_v(j >> 1, p.L, h);
        s0[i & 1] += f[i];
        sz = fma(vz, f[i], sz);
        szz = fma(vz * vz, f[i], szz);
      }
#pragma unroll
      for (int cch = 0; cch < CPB; ++cch) {
        double g[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) g[i] = f[16 * cch + i];
        tm_st16(taddr + (bb + cch) * 32, g);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    const double sall = s0[0] + s0[1];
    double m[5] = {sall, vx * sall, vy[0] * s0[0] + vy[1] * s0[1], sz,
                   vx * vx * sall + (vy[0] * vy[0] * s0[0] + vy[1] * vy[1] * s0[1]) + szz};
    block_sum5<NT>(m, red);
    double U[5] = {m[0], m[1], m[2], m[3], m[4]};
    const double rho = vol * m[0];
    double u[3], uu = 0.0;
    for (int a = 0; a < DV; ++a) {
      u[a] = vol * m[1 + a] / rho;
      uu += u[a] * u[a];
    }
    const double T = (vol * m[4] / rho - uu) / DV;
    const double amp = rho / pow(2.0 * 3.141592653589793 * T, 0.5 * DV);
    if (t < DV * N) {
      const int a = t / N, k = t % N;
      const double wv = node_v(k, p.L, h) - u[a];
      sexp[a][k] = exp(-(wv * wv) / (2.0 * T));
    }
    __syncthreads();
    double S0[3], S1[3], S2[3];
    for (int a = 0; a < DV; ++a) {
      double q0 = 0.0, q1 = 0.0, q2 = 0.0;
      for (int k = 0; k < N; ++k) {
        const double e = sexp[a][k], v = node_v(k, p.L, h);
        q0 += e;
        q1 = fma(v, e, q1);
        q2 = fma(v * v, e, q2);
      }
      S0[a] = q0;
      S1[a] = q1;
      S2[a] = q2;
    }
    double me[5];
    me[0] = amp * S0[0] * S0[1] * S0[2];
    me[1] = amp * S1[0] * S0[1] * S0[2];
    me[2] = amp * S0[0] * S1[1] * S0[2];
    me[3] = amp * S0[0] * S0[1] * S1[2];
    me[4] = amp * (S2[0] * S0[1] * S0[2] + S0[0] * S2[1] * S0[2] + S0[0] * S0[1] * S2[2]);
    double lam[5];
    for (int a = 0; a < NM; ++a) {
      double sacc = 0.0;
      for (int b = 0; b < NM; ++b) sacc = fma(p.Ginv[a * NM + b], U[b] - me[b], sacc);
      lam[a] = sacc;
    }
    const double nu = p.nu_rule == 0 ? rho : p.mu;
    const double c1 = p.dt_tau * nu;
    // E(k) = amp e_x e_y e_z + lam0 + lam1 vx + lam2 vy + lam3 vz + lam4 |v|^2: the x/y parts per parity
    double exy[2], cst[2];
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      exy[par] = amp * sexp[0][kx] * sexp[1][ky0 + 16 * par];
      cst[par] = lam[0] + lam[1] * vx + lam[2] * vy[par] + lam[4] * (vx * vx + vy[par] * vy[par]);
    }
    bool bad = false;
    double* out = p.f_out + cell * n;
#pragma unroll 1
    for (int b = 0; b < NB; ++b) {  // pass 3: f* from TMEM, E = E~ + Phi^T lambda, Euler
      double f[16];
      tm_ld16(taddr + b * 32, f);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = 16 * b + i;
        const int kz = j >> 1, par = i & 1;
        const double vz = node_v(kz, p.L, h);
        const double E = fma(exy[par], sexp[2][kz], fma(lam[4], vz * vz, fma(lam[3], vz, cst[par])));
        const double o = p.nu_rule == 2 ? E : fma(c1, E - f[i], f[i]);
        bad |= !isfinite(o);
        out[t + NT * j] = o;
      }
    }
    if (bad) atomicOr(p.nonfinite, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_slot), "n"(512) : "memory");
}

// 2D cells (N^2 <= 1024 nodes): one warp per cell, homogeneous (dx = 0) only; reductions are
// warp shuffles in a fixed order.  Same arithmetic as k_bgk.
template <int N, int MINB>
__global__ void __launch_bounds__(256, MINB) k_bgk2w(const BgkParams p) {
  constexpr int n = N * N;
  __shared__ double sexp[8][2][N];
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  const double h = p.dv, vol = h * h;
  for (int it = blockIdx.x * 8 + wv; it < p.ncells; it += gridDim.x * 8) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const double2* src = reinterpret_cast<const double2*>(p.f_in + cell * n);
    double m[5] = {0, 0, 0, 0, 0};
#pragma unroll 4
    for (int k2 = lane; k2 < n / 2; k2 += 32) {
      const double2 f2 = __ldg(src + k2);
      double ph[5], pq[5];
      phi_row<N, 2>(2 * k2, p.L, h, ph);
      phi_row<N, 2>(2 * k2 + 1, p.L, h, pq);
#pragma unroll
      for (int c = 0; c < 5; ++c) m[c] = fma(pq[c], f2.y, fma(ph[c], f2.x, m[c]));
    }
#pragma unroll
    for (int c = 0; c < 5; ++c) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) m[c] += __shfl_xor_sync(0xffffffffu, m[c], o);
    }
    const double rho = vol * m[0];
    const double u0 = vol * m[1] / rho, u1 = vol * m[2] / rho;
    const double T = (vol * m[4] / rho - (u0 * u0 + u1 * u1)) / 2;
    const double amp = rho / pow(2.0 * 3.141592653589793 * T, 1.0);
    __syncwarp();
    for (int i = lane; i < 2 * N; i += 32) {
      const int a = i / N, k = i % N;
      const double w = node_v(k, p.L, h) - (a == 0 ? u0 : u1);
      sexp[wv][a][k] = exp(-(w * w) / (2.0 * T));
    }
    __syncwarp();
    auto maxw = [&](int k) { return amp * sexp[wv][0][k % N] * sexp[wv][1][k / N]; };
    // separable moments of E~ (as in k_bgk)
    double S0[2], S1[2], S2[2];
    for (int a = 0; a < 2; ++a) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int k = 0; k < N; ++k) {
        const double e = sexp[wv][a][k], v = node_v(k, p.L, h);
        s0 += e;
        s1 = fma(v, e, s1);
        s2 = fma(v * v, e, s2);
      }
      S0[a] = s0;
      S1[a] = s1;
      S2[a] = s2;
    }
    const double me[5] = {amp * S0[0] * S0[1], amp * S1[0] * S0[1], amp * S0[0] * S1[1], 0.0,
                          amp * (S2[0] * S0[1] + S0[0] * S2[1])};
    const double r[4] = {m[0] - me[0], m[1] - me[1], m[2] - me[2], m[4] - me[4]};
    double lam[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double sacc = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) sacc = fma(p.Ginv[a * 4 + b], r[b], sacc);
      lam[a] = sacc;
    }
    const double c1 = p.dt_tau * (p.nu_rule == 0 ? rho : p.mu);
    bool bad = false;
    auto update = [&](int k, double f) {
      double ph[5];
      phi_row<N, 2>(k, p.L, h, ph);
      double E = maxw(k) + lam[0];
      E = fma(lam[1], ph[1], E);
      E = fma(lam[2], ph[2], E);
      E = fma(lam[3], ph[4], E);
      const double o = p.nu_rule == 2 ? E : fma(c1, E - f, f);
      bad |= !isfinite(o);
      return o;
    };
    double2* dst = reinterpret_cast<double2*>(p.f_out + cell * n);
#pragma unroll 4
    for (int k2 = lane; k2 < n / 2; k2 += 32) {
      const double2 f2 = __ldg(src + k2);
      const double o0 = update(2 * k2, f2.x), o1 = update(2 * k2 + 1, f2.y);
      dst[k2] = make_double2(o0, o1);
    }
    if (bad) atomicOr(p.nonfinite, 1);
  }
}

cudaError_t launch_bgk(int N, int dv, const BgkParams& p, int sm_count, cudaStream_t s) {
  if (p.ncells == 0) return cudaSuccess;
  if (dv == 2 && p.tp.dx == 0) {
    // FKS_BGK2_CFG (experiment knob): resident CTAs per SM the register cap aims at (1, 3 or 4);
    // 3 (80 registers) measured best at the C1 shape (profiles/r01_optimisation_log.md)
    static const int minb = [] {  // read once
      const char* e = getenv("FKS_BGK2_CFG");
      return e ? atoi(e) : 3;
    }();
    const int per_sm = minb == 1 ? 8 : 2 * minb;
    const unsigned nw = (unsigned)((p.ncells + 7) / 8 < sm_count * per_sm ? (p.ncells + 7) / 8 : sm_count * per_sm);
#define FKS_BGK2(NN)                                                        \
    if (N == NN) {                                                          \
      if (minb == 4) k_bgk2w<NN, 4><<<nw, 256, 0, s>>>(p);                  \
      else if (minb == 3) k_bgk2w<NN, 3><<<nw, 256, 0, s>>>(p);             \
      else k_bgk2w<NN, 1><<<nw, 256, 0, s>>>(p);                            \
      return cudaGetLastError();                                            \
    }
    FKS_BGK2(8) FKS_BGK2(16) FKS_BGK2(32)
#undef FKS_BGK2
  }
  // 3D cells are 256 KiB: CTAs per SM x 148 x 256 KiB (x2 with the next-cell prefetch) must fit
  // the 126 MB L2, or pass 3 re-reads f from HBM.  FKS_BGK_CFG (experiment knob) = 0: 256 threads x
  // 8 CTAs/SM + prefetch (the round-1 launch); 2: 512 x 2, no prefetch; 3: 512 x 1 + prefetch;
  // 4: 512 x 2 capped at 64 registers (2 resident), no prefetch; 5: 256 x 4 at 64 registers.
  static const int cfg_env = [] {  // read once; -1: not set
    const char* e = getenv("FKS_BGK_CFG");
    return e ? atoi(e) : -1;
  }();
  int cfg = cfg_env >= 0 ? cfg_env : (dv == 3 && N == 32) ? 6 : 0;
  if (cfg == 6 && dv == 3 && N == 32) {  // f* in TMEM: one 512-thread CTA per SM (all TMEM columns)
    const unsigned nb6 = (unsigned)(p.ncells < sm_count ? p.ncells : sm_count);
    static const bool bw32 = [] {  // experiment knob: gathers in flight per thread (read once)
      const char* e = getenv("FKS_BGK_BW");
      return e && atoi(e) == 32;
    }();
    if (bw32) k_bgk_tmem32<32><<<nb6, 512, 0, s>>>(p);
    else k_bgk_tmem32<16><<<nb6, 512, 0, s>>>(p);
    return cudaGetLastError();
  }
  if (cfg == 6) cfg = 0;
  const int per_sm = cfg == 0 ? 8 : (cfg == 2 || cfg == 4) ? 2 : cfg == 5 ? 4 : 1;
  const int pf = (cfg == 0 || cfg == 3) ? 1 : 0;
  const unsigned nb = (unsigned)(p.ncells < sm_count * per_sm ? p.ncells : sm_count * per_sm);
#define FKS_BGK(NN, DD)                                                                      \
  if (N == NN && dv == DD) {                                                                 \
    if (cfg == 4) k_bgk<NN, DD, 512, 2><<<nb, 512, 0, s>>>(p, pf);                           \
    else if (cfg == 5) k_bgk<NN, DD, 256, 4><<<nb, 256, 0, s>>>(p, pf);                      \
    else if (cfg == 2 || cfg == 3) k_bgk<NN, DD, 512, 1><<<nb, 512, 0, s>>>(p, pf);           \
    else k_bgk<NN, DD, 256, 1><<<nb, 256, 0, s>>>(p, pf);                                    \
    return cudaGetLastError();                                                               \
  }
  FKS_BGK(4, 2) FKS_BGK(8, 2) FKS_BGK(16, 2) FKS_BGK(32, 2) FKS_BGK(64, 2) FKS_BGK(4, 3) FKS_BGK(8, 3) FKS_BGK(16, 3) FKS_BGK(32, 3) FKS_BGK(64, 3)
#undef FKS_BGK
  return cudaErrorInvalidValue;
}

}  // namespace fks
