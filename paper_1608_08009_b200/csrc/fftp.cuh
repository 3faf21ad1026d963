// Pencil FFTs of length N (<= 64) split over a lane pair (h = lane & 1 owns N/2 complex values),
// one radix-2 stage across the pair through shuffles, the N/2-point remainders in registers
// (fft.cuh).  Used by kernels2dp.cu (2D, N = 32 / 64) and kernels3d64.cu (3D, N = 64).
//   forward (DIF): thread h holds x[N/2 h + j] (halves) -> thread h gets X[2m + h] (parity);
//   inverse (DIT): thread h holds x[2m + h] (parity) -> thread h gets X[N/2 h + j] (halves).
#pragma once
#include "fft.cuh"

namespace fks {

__device__ __forceinline__ double2 shfl_pair(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 1), __shfl_xor_sync(0xffffffffu, v.y, 1));
}

// x * exp(SIGN 2 pi i kk / 64) if `on`, else x (kk compile-time after unrolling).
template <int SIGN>
__device__ __forceinline__ double2 twiddle_if(double2 x, int kk, bool on) {
  const double2 t = twiddle<SIGN>(x, kk);
  return on ? t : x;
}

// DIF: a[j] = x[H h + j] -> a[m] = X[2m + h]  (X_k = sum_j x_j exp(SIGN 2 pi i j k / N))
template <int N, int SIGN>
__device__ __forceinline__ void fftp_dif(double2 (&a)[N / 2], int h) {
  const double sg = h ? -1.0 : 1.0;
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    const double2 b = shfl_pair(a[j]);
    // h = 0: x_j + x_{j+H};  h = 1: (x_j - x_{j+H}) W_N^j  (b is the partner's value)
    const double2 u = make_double2(b.x + sg * a[j].x, b.y + sg * a[j].y);
    a[j] = twiddle_if<SIGN>(u, j * (64 / N), h != 0);
  }
  fft<N / 2, SIGN>(a);
}

// DIT: a[m] = x[2m + h] -> a[j] = X[H h + j]
template <int N, int SIGN>
__device__ __forceinline__ void fftp_dit(double2 (&a)[N / 2], int h) {
  fft<N / 2, SIGN>(a);  // h = 0: E_k (even inputs), h = 1: O_k (odd inputs)
  const double sg = h ? -1.0 : 1.0;
#pragma unroll
  for (int k = 0; k < N / 2; ++k) {
    const double2 t = twiddle_if<SIGN>(a[k], k * (64 / N), h != 0);  // h = 1: W^k O_k
    const double2 b = shfl_pair(t);
    // h = 0: X_k = E_k + W^k O_k;  h = 1: X_{k+H} = E_k - W^k O_k
    a[k] = make_double2(b.x + sg * t.x, b.y + sg * t.y);
  }
}

}  // namespace fks
