// 2D fused collision / step kernel (a3-a9) for Maxwell molecules on an N^2 velocity grid.
//
// A group of N threads owns one cell (several groups per CTA, persistent over cells).  The
// whole cell lives in SMEM: f^ (N^2 complex) and one N^2 work plane (rows padded to N+1 to
// keep row and column sweeps bank-conflict free).  Per direction p:
//   column pass: thread l_x forms X = (alpha~_p + i alpha'~_p) f^ along l_y and IFFTs it,
//   row pass:    thread j_y IFFTs its row and accumulates G[j_y][.] += Re z Im z in registers.
// The loss is the (A+1)-th direction with table (D~, 0).  Thread j_y then owns row j_y of Q for
// the projection (a group reduction of 4 moments) and the Euler update.
// Folded tables: T[p][l_y][l_x] double2 = (s w_p alpha_p / n, alpha'_p / n); T[A] = (s D / n, 0).
#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace fks {

template <int N>
struct Cfg2 {
  static constexpr int RS = N + 1;
  static constexpr int GROUPS = N == 32 ? 6 : 8;   // cells per CTA
  static constexpr int THREADS = GROUPS * N;
  static constexpr size_t PER_GROUP = (size_t)N * N * 16 + (size_t)N * RS * 16;
  static constexpr size_t SMEM = GROUPS * PER_GROUP + 3 * kMaxN;  // + int8 shift table
};

template <int N>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = N / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(mask, v, o, N);
  return v;
}

template <int N>
__global__ void __launch_bounds__(Cfg2<N>::THREADS, 1) k_step2d(const StepParams p) {
  using C = Cfg2<N>;
  constexpr int RS = C::RS;
  constexpr int n = N * N;
  extern __shared__ __align__(128) unsigned char smem[];
  const int g = threadIdx.x / N;
  const int tx = threadIdx.x % N;
  double2* fhat = reinterpret_cast<double2*>(smem + g * C::PER_GROUP);  // [l_y][l_x]
  double2* wk = fhat + n;                                               // [y][RS]
  const unsigned lane = threadIdx.x & 31;
  const unsigned mask = N >= 32 ? 0xffffffffu : (((1u << N) - 1u) << (lane & ~(unsigned)(N - 1)));
  const int ngroups = gridDim.x * C::GROUPS;
  int8_t (*sdelta)[kMaxN] = reinterpret_cast<int8_t (*)[kMaxN]>(smem + C::GROUPS * C::PER_GROUP);
  load_delta(p.tp, sdelta);
  __syncthreads();

  for (int it = blockIdx.x * C::GROUPS + g; it < p.ncells; it += ngroups) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    const CellCoord cc = cell_coord(p.tp, cell);
    // a3: row y = tx of f*, forward FFT along x
    {
      double2 r[N];
#pragma unroll
      for (int x = 0; x < N; ++x)
        r[x] = make_double2(gather_fstar(p.f_in, p.tp, cc, x + N * tx, x, tx, 0, n, sdelta), 0.0);
      fft<N, -1>(r);
#pragma unroll
      for (int x = 0; x < N; ++x) wk[tx * RS + x] = r[x];
    }
    __syncwarp(mask);
    {
      double2 c[N];
#pragma unroll
      for (int y = 0; y < N; ++y) c[y] = wk[y * RS + tx];
      fft<N, -1>(c);
#pragma unroll
      for (int ly = 0; ly < N; ++ly) fhat[ly * N + tx] = c[ly];
    }
    __syncwarp(mask);
    double gacc[N];
#pragma unroll
    for (int x = 0; x < N; ++x) gacc[x] = 0.0;
#pragma unroll 1
    for (int d = 0; d <= p.A; ++d) {
      {
        double2 c[N];
        const double2* T = p.tables + (size_t)d * n + tx;
#pragma unroll
        for (int ly = 0; ly < N; ++ly) {
          const double2 t = __ldg(T + ly * N), F = fhat[ly * N + tx];
          c[ly] = make_double2(fma(t.x, F.x, -t.y * F.y), fma(t.x, F.y, t.y * F.x));
        }
        fft<N, +1>(c);
#pragma unroll
        for (int y = 0; y < N; ++y) wk[y * RS + tx] = c[y];
      }
      __syncwarp(mask);
      {
        double2 r[N];
#pragma unroll
        for (int x = 0; x < N; ++x) r[x] = wk[tx * RS + x];
        fft<N, +1>(r);
        if (d < p.A) {
#pragma unroll
          for (int x = 0; x < N; ++x) gacc[x] = fma(r[x].x, r[x].y, gacc[x]);
        } else {
#pragma unroll
          for (int x = 0; x < N; ++x) {
            const double fs = gather_fstar(p.f_in, p.tp, cc, x + N * tx, x, tx, 0, n, sdelta);
            gacc[x] = gacc[x] - fs * r[x].x;  // gacc now holds Q
          }
        }
      }
      __syncwarp(mask);
    }
    double* out = p.f_out + cell * (int64_t)n;
    const double* q = gacc;
    if (p.mode == 0) {
#pragma unroll
      for (int x = 0; x < N; ++x) out[x + N * tx] = q[x];
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
#pragma unroll
    for (int x = 0; x < N; ++x) {
      const double vx = node_v(x, p.L, p.dv);
      const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * (vx * vx + vy * vy);
      const double fs = gather_fstar(p.f_in, p.tp, cc, x + N * tx, x, tx, 0, n, sdelta);
      const double o = fma(p.dt_tau, q[x] - corr, fs);
      bad |= !isfinite(o);
      out[x + N * tx] = o;
    }
    if (bad) atomicOr(p.nonfinite, 1);
  }
}

template <int N>
static cudaError_t launch2(const StepParams& p, int nblocks, cudaStream_t s) {
  using C = Cfg2<N>;
  cudaError_t e = cudaFuncSetAttribute(k_step2d<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) return e;
  k_step2d<N><<<nblocks, C::THREADS, C::SMEM, s>>>(p);
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

}  // namespace fks
