// Register-resident radix-2^2 FFTs of length 8/16/32 in fp64 for sm_100a.
//
// The paper evaluates its A convolutions with "standard FFT technique" (FFTW 3.3.4 in
// its runs).  Here one thread owns one whole 1D pencil in registers; the compiler
// fully unrolls the butterflies and every twiddle is an immediate operand (trivial twiddles
// 1, -1, +-i and (+-1 +- i)/sqrt2 are special-cased), so a 32-point transform is ~450 DP
// instructions with no shared-memory traffic.  Twiddles are exact fp64 constants
// cos(2 pi k / 64) (no recurrences; DESIGN.md "parity" notes).
#pragma once
#include <cuda_runtime.h>

namespace fks {

// cos(2 pi k / 64), k = 0..16 (quarter wave), correctly rounded.
__device__ __forceinline__ constexpr double cos64q(int k) {
  constexpr double t[17] = {
      1.00000000000000000e+00, 9.95184726672196929e-01, 9.80785280403230431e-01,
      9.56940335732208824e-01, 9.23879532511286738e-01, 8.81921264348355050e-01,
      8.31469612302545236e-01, 7.73010453362736993e-01, 7.07106781186547573e-01,
      6.34393284163645488e-01, 5.55570233019602289e-01, 4.71396736825997809e-01,
      3.82683432365089837e-01, 2.90284677254462331e-01, 1.95090322016128331e-01,
      9.80171403295607702e-02, 0.0};
  return t[k];
}

__device__ __forceinline__ constexpr double cos64(int k) {
  k &= 63;
  return k <= 16 ? cos64q(k) : k <= 32 ? -cos64q(32 - k) : k <= 48 ? -cos64q(k - 32) : cos64q(64 - k);
}

__device__ __forceinline__ constexpr double sin64(int k) { return cos64(k - 16); }

// x * exp(SIGN * 2 pi i kk / 64); kk is a compile-time constant after unrolling.
template <int SIGN>
__device__ __forceinline__ double2 twiddle(double2 x, int kk) {
  kk &= 63;
  if (kk == 0) return x;
  if (kk == 32) return make_double2(-x.x, -x.y);
  if (kk == 16) return SIGN > 0 ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
  if (kk == 48) return SIGN > 0 ? make_double2(x.y, -x.x) : make_double2(-x.y, x.x);
  const double c = cos64(kk);
  const double s = SIGN > 0 ? sin64(kk) : -sin64(kk);
  if ((kk & 7) == 0) {  // |c| = |s| = sqrt(1/2)
    if (s == c) return make_double2(c * (x.x - x.y), c * (x.x + x.y));
    return make_double2(c * (x.x + x.y), c * (x.y - x.x));
  }
  return make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c));
}

template <int N>
__device__ __forceinline__ constexpr int bitrev(int j) {
  int r = 0;
  for (int b = 1; b < N; b <<= 1) {
    r <<= 1;
    if (j & b) r |= 1;
  }
  return r;
}

// In-place DFT of length N (power of two, <= 64): x_j <- sum_k x_k exp(SIGN 2 pi i j k / N).
// Unnormalised in both directions.  Radix-2^2 decimation in frequency: two radix-2 stages are
// fused per block of M points (quarter Q = M/4) so the inner twiddle is the free +-i and only
// three twiddles W_M^{2k}, W_M^{k}, W_M^{3k} remain (four in plain radix-2); the data flow and
// hence the bit-reversed output order are those of radix-2 DIF.  A final radix-2 stage handles
// odd log2 N.
// hook(h) is called before each radix-4 stage, before the final radix-2 stage (if any) and after
// the last stage (h = 0, 1, ...): callers interleave independent memory work with the butterflies.
template <int N, int SIGN, typename Hook>
__device__ __forceinline__ void fft_hooked(double2 (&x)[N], Hook&& hook) {
  int h = 0;
#pragma unroll
  for (int M = N; M >= 4; M >>= 2) {
    hook(h++);
    const int Q = M / 4;
#pragma unroll
    for (int start = 0; start < N; start += M) {
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        const double2 a0 = x[start + k], a1 = x[start + k + Q], a2 = x[start + k + 2 * Q],
                      a3 = x[start + k + 3 * Q];
        const double2 u0 = make_double2(a0.x + a2.x, a0.y + a2.y);
        const double2 u2 = make_double2(a0.x - a2.x, a0.y - a2.y);
        const double2 u1 = make_double2(a1.x + a3.x, a1.y + a3.y);
        const double2 d13 = make_double2(a1.x - a3.x, a1.y - a3.y);
        // u3 = (a1 - a3) * (SIGN i)
        const double2 u3 = SIGN > 0 ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
        x[start + k] = make_double2(u0.x + u1.x, u0.y + u1.y);
        const int step = 64 / M;
        x[start + k + Q] = twiddle<SIGN>(make_double2(u0.x - u1.x, u0.y - u1.y), 2 * k * step);
        x[start + k + 2 * Q] = twiddle<SIGN>(make_double2(u2.x + u3.x, u2.y + u3.y), k * step);
        x[start + k + 3 * Q] = twiddle<SIGN>(make_double2(u2.x - u3.x, u2.y - u3.y), 3 * k * step);
      }
    }
    if (M / 4 == 2) {  // one radix-2 stage left (log2 N odd)
      hook(h++);
#pragma unroll
      for (int start = 0; start < N; start += 2) {
        const double2 a = x[start], b = x[start + 1];
        x[start] = make_double2(a.x + b.x, a.y + b.y);
        x[start + 1] = make_double2(a.x - b.x, a.y - b.y);
      }
    }
  }
  hook(h++);
  double2 y[N];
#pragma unroll
  for (int j = 0; j < N; ++j) y[j] = x[bitrev<N>(j)];
#pragma unroll
  for (int j = 0; j < N; ++j) x[j] = y[j];
}

template <int N, int SIGN>
__device__ __forceinline__ void fft(double2 (&x)[N]) {
  fft_hooked<N, SIGN>(x, [](int) {});
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

}  // namespace fks
