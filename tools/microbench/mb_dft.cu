// NEXT-4 tensor-core gate (north_star: "small-N DFT stages go on tensor cores only if
// ncu shows it beats the FFT path"): 32-point complex DFTs per second on one B200,
//   (a) the register FFT of the hot kernels (fks::fft<32>, fft.cuh), one pencil per thread;
//   (b) the same DFTs as dense fp64 matrix products on the tensor pipe: X = W x with W the 32 x 32
//       DFT matrix, mma.sync.m8n8k4.f64 (DMMA), 8 pencils per warp tile, complex as 4 real products,
//       W fragments held in registers.
// fp64 has no tcgen05 kind, so DMMA is the only fp64 tensor instruction.  Both paths are checked
// against each other (max relative difference printed) and timed with CUDA events, compute-bound
// (data kept in registers, R repetitions).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1608_08009_b200/csrc -o mb_dft mb_dft.cu
#include <cmath>
#include <cstdio>
#include <vector>

#include "fft.cuh"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int R = 64;  // repetitions per launch (compute-bound)

// (a) register FFT: per repetition a forward and an inverse 32-point transform and the 1/32 scale
__global__ void k_fft(const double2* in, double2* out, int reps) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double2 x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = in[(size_t)t * 32 + j];
  for (int r = 0; r < reps; ++r) {
    fks::fft<32, +1>(x);
    fks::fft<32, -1>(x);
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = make_double2(x[j].x * (1.0 / 32), x[j].y * (1.0 / 32));
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) out[(size_t)t * 32 + j] = x[j];
}

// one forward DFT of each pencil with the register FFT (reference for the DMMA path)
__global__ void k_fft_once(const double2* in, double2* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double2 x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = in[(size_t)t * 32 + j];
  fks::fft<32, +1>(x);
#pragma unroll
  for (int j = 0; j < 32; ++j) out[(size_t)t * 32 + j] = x[j];
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// (b) DMMA: a warp transforms 8 pencils (columns of x); fragment layouts of m8n8k4.f64:
// A (8 x 4): a = A[lane >> 2][lane & 3]; B (4 x 8): b = B[lane & 3][lane >> 2];
// C (8 x 8): c0, c1 = C[lane >> 2][2 (lane & 3) + {0, 1}].
// X = W x, W_jk = exp(+2 pi i j k / 32): row tile t (outputs 8t..8t+7), k-step s (inputs 4s..4s+3).
__global__ void k_dmma(const double2* in, double2* out, int reps) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  double wr[4][8], wi[4][8], wn[4][8];  // W fragments (re, im, -im) per (t, s)
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int j = 8 * t + ar, k = 4 * s + ac;
      double sn, cs;
      sincospi(2.0 * ((j * k) % 32) / 32.0, &sn, &cs);
      wr[t][s] = cs;
      wi[t][s] = sn;
      wn[t][s] = -sn;
    }
  // B fragments: x[4s + (lane & 3)][pencil lane >> 2] of this warp's 8 pencils
  double xr[8], xi[8];
  const size_t p = (size_t)warp * 8 + (lane >> 2);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const double2 v = in[p * 32 + 4 * s + (lane & 3)];
    xr[s] = v.x;
    xi[s] = v.y;
  }
  // the accumulators run on across the repetitions (the result is reps x the DFT), so every
  // repetition's products are live: a loop-invariant product would otherwise be hoisted by the
  // compiler (an earlier version measured a phantom 400 TF/s that way; ncu counted the instructions)
  double cr[4][2] = {}, ci[4][2] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        dmma(cr[t][0], cr[t][1], wr[t][s], xr[s]);  // Re += Wr xr
        dmma(cr[t][0], cr[t][1], wn[t][s], xi[s]);  // Re -= Wi xi
        dmma(ci[t][0], ci[t][1], wr[t][s], xi[s]);  // Im += Wr xi
        dmma(ci[t][0], ci[t][1], wi[t][s], xr[s]);  // Im += Wi xr
      }
    }
  }
  const double sc = 1.0 / reps;
  // C[row = output j][col = pencil]: thread holds outputs 8t + (lane >> 2), pencils 2 (lane & 3) + {0, 1}
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const size_t pc = (size_t)warp * 8 + 2 * (lane & 3) + e;
      out[pc * 32 + 8 * t + (lane >> 2)] = make_double2(cr[t][e] * sc, ci[t][e] * sc);
    }
}

// round-1 style: 4 dependent accumulator chains per warp (latency-bound)
__global__ void k_dmma_chain(double* out, int iters) {
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.5;
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dmma(c0, c1, a, b); dmma(d0, d1, a, b); dmma(e0, e1, a, b); dmma(f0, f1, a, b);
    }
  }
  double s = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1;
  if (s == 12345.678) out[0] = s;
}

// many independent accumulators per warp (throughput-bound)
__global__ void k_dmma_wide(double* out, int iters) {
  double a = threadIdx.x * 1e-9 + 1.0, b = 0.5;
  double c[16][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int threads = 256;
  const int blocks = sms * 8;
  const size_t pencils = (size_t)blocks * threads;  // (a): one per thread; (b): 8 per warp
  std::vector<double2> h(pencils * 32);
  unsigned s = 12345;
  for (auto& v : h) {
    s = s * 1664525u + 1013904223u;
    v.x = (s >> 8) / 16777216.0 - 0.5;
    s = s * 1664525u + 1013904223u;
    v.y = (s >> 8) / 16777216.0 - 0.5;
  }
  double2 *din, *dout, *dref;
  CK(cudaMalloc(&din, h.size() * 16));
  CK(cudaMalloc(&dout, h.size() * 16));
  CK(cudaMalloc(&dref, h.size() * 16));
  CK(cudaMemcpy(din, h.data(), h.size() * 16, cudaMemcpyHostToDevice));
  // correctness: one DMMA DFT vs one register FFT of the first pencils
  const size_t dmma_pencils = (size_t)blocks * threads / 32 * 8;
  k_fft_once<<<blocks, threads>>>(din, dref);
  k_dmma<<<blocks, threads>>>(din, dout, 1);
  CK(cudaDeviceSynchronize());
  std::vector<double2> a(dmma_pencils * 32), b(dmma_pencils * 32);
  CK(cudaMemcpy(a.data(), dref, a.size() * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), dout, b.size() * 16, cudaMemcpyDeviceToHost));
  double err = 0, mx = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    err = fmax(err, fmax(fabs(a[i].x - b[i].x), fabs(a[i].y - b[i].y)));
    mx = fmax(mx, fmax(fabs(a[i].x), fabs(a[i].y)));
  }
  printf("DMMA DFT vs register FFT, %zu pencils: max |diff| / max |X| = %.2e\n", dmma_pencils, err / mx);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int round = 0; round < 2; ++round) {
    float ms;
    k_fft<<<blocks, threads>>>(din, dout, R);
    cudaEventRecord(e0);
    k_fft<<<blocks, threads>>>(din, dout, R);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double fft_rate = (double)pencils * R * 2 / (ms * 1e-3);  // 2 transforms per repetition
    k_dmma<<<blocks, threads>>>(din, dout, R);
    CK(cudaGetLastError());
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(din, dout, R);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma_rate = (double)dmma_pencils * R / (ms * 1e-3);
    {  // the timed launch computed the same transforms
      std::vector<double2> c(b.size());
      CK(cudaMemcpy(c.data(), dout, c.size() * 16, cudaMemcpyDeviceToHost));
      double d2 = 0;
      for (size_t i = 0; i < c.size(); ++i) d2 = fmax(d2, fmax(fabs(c[i].x - a[i].x), fabs(c[i].y - a[i].y)));
      printf("  timed DMMA launch (sum of %d repetitions / %d) vs FFT: max |diff| / max |X| = %.2e (%.3f ms)\n", R, R, d2 / mx, ms);
    }
    printf("round %d: register FFT %.3e 32-point DFTs/s (%.1f TFLOP/s in the 5 N log2 N convention); "
           "DMMA dense DFT %.3e DFTs/s (%.1f TFLOP/s of 8 N^2 matrix flops) -> FFT / DMMA = %.1fx\n",
           round, fft_rate, fft_rate * 5 * 32 * 5 / 1e12, dmma_rate, dmma_rate * 8.0 * 32 * 32 / 1e12,
           fft_rate / dmma_rate);
  }
  for (int reps : {16, 64, 256}) {  // the DMMA DFT time must scale with the repetitions
    float ms;
    k_dmma<<<blocks, threads>>>(din, dout, reps);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(din, dout, reps);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA DFT reps %3d: %.4f ms\n", reps, ms);
  }
  {
    double* o;
    CK(cudaMalloc(&o, 8));
    const int iters = 4096;
    float ms;
    for (int tpb : {128, 256, 512}) {
      k_dmma_chain<<<sms * 4, tpb>>>(o, 16);
      cudaEventRecord(e0);
      k_dmma_chain<<<sms * 4, tpb>>>(o, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      const double chain = 512.0 * 32 * iters * (double)sms * 4 * tpb / 32 / (ms * 1e-3) / 1e12;
      k_dmma_wide<<<sms * 4, tpb>>>(o, 16);
      cudaEventRecord(e0);
      k_dmma_wide<<<sms * 4, tpb>>>(o, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      const double wide = 512.0 * 16 * iters * (double)sms * 4 * tpb / 32 / (ms * 1e-3) / 1e12;
      printf("DMMA m8n8k4 peak, %d threads x %d CTAs: 4 dependent chains %.1f TFLOP/s, 16 independent %.1f TFLOP/s\n",
             tpb, sms * 4, chain, wide);
    }
  }
  return 0;
}
