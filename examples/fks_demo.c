/*
 * fks_demo.c -- the C ABI used from plain C (no Python): a batch of homogeneous 3D cells relaxing
 * from two-Maxwellian states (the shape of the paper's Test 1.3 relaxation), ten fused
 * steps (a4..a9) with fks_step, the moments (a10) after every step.  Mass, momentum and energy are
 * conserved by the projection to round-off; the temperature anisotropy (T_xx > T)
 * relaxes toward T.
 *
 *   gcc -std=c11 -O2 examples/fks_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1608_08009_b200 -lfks -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1608_08009_b200 -lm -o fks_demo && ./fks_demo
 *
 * Exit status 0 when every call succeeded and the conservation checks hold.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "fks.h"

#define CHECK(call)                                                                           \
  do {                                                                                        \
    fks_status s_ = (call);                                                                   \
    if (s_ != FKS_OK) {                                                                       \
      fprintf(stderr, "%s failed: %s\n", #call, fks_strerror(s_));                           \
      return 1;                                                                               \
    }                                                                                         \
  } while (0)

#define CUDA(call)                                                                            \
  do {                                                                                        \
    if ((call) != cudaSuccess) {                                                              \
      fprintf(stderr, "%s failed\n", #call);                                                  \
      return 1;                                                                               \
    }                                                                                         \
  } while (0)

static const double kPi = 3.14159265358979323846;

/* directional temperature T_xx = int (v_x - u_x)^2 f / rho of one cell (host copy) */
static double txx(const double* f, int N, double L, double ux) {
  const double h = 2.0 * L / N;
  double m0 = 0.0, m2 = 0.0;
  for (int k = 0; k < N * N * N; ++k) {
    const double vx = -L + (k % N + 0.5) * h - ux;
    m0 += f[k];
    m2 += vx * vx * f[k];
  }
  return m2 / m0;
}

static double u2(const double* u, int c) { return u[3 * c] * u[3 * c] + u[3 * c + 1] * u[3 * c + 1] + u[3 * c + 2] * u[3 * c + 2]; }

int main(void) {
  const int N = 16, cells = 64, steps = 10;
  const double L = 7.0, dt = 0.05;
  const int n = N * N * N;
  const double h = 2.0 * L / N;
  fks_grid grid = {0};
  grid.dv = 3;
  grid.dx = 0;
  grid.M[0] = cells;
  grid.h = 1.0;
  fks_ctx* ctx = NULL;
  CHECK(fks_init(&grid, N, L, 24, 1.0, &ctx));  /* hard spheres, the 24-point spherical design */
  CHECK(fks_set_params(ctx, 1.0, 0.0, 0.0, 1)); /* tau = 1, default kernel constant and R */

  /* f = two Maxwellians displaced along x, cell c with separation 1 + c / cells */
  double* f = (double*)malloc((size_t)cells * n * sizeof(double));
  for (int c = 0; c < cells; ++c) {
    const double a = 1.0 + (double)c / cells;
    for (int k = 0; k < n; ++k) {
      const double vx = -L + (k % N + 0.5) * h, vy = -L + ((k / N) % N + 0.5) * h;
      const double vz = -L + (k / (N * N) + 0.5) * h;
      const double r2 = vy * vy + vz * vz;
      f[(size_t)c * n + k] = 0.5 / pow(2.0 * kPi, 1.5) *
                             (exp(-0.5 * ((vx - a) * (vx - a) + r2)) + exp(-0.5 * ((vx + a) * (vx + a) + r2)));
    }
  }
  double *d_a, *d_b, *d_rho, *d_u, *d_T;
  CUDA(cudaMalloc((void**)&d_a, (size_t)cells * n * sizeof(double)));
  CUDA(cudaMalloc((void**)&d_b, (size_t)cells * n * sizeof(double)));
  CUDA(cudaMalloc((void**)&d_rho, cells * sizeof(double)));
  CUDA(cudaMalloc((void**)&d_u, 3 * cells * sizeof(double)));
  CUDA(cudaMalloc((void**)&d_T, cells * sizeof(double)));
  CUDA(cudaMemcpy(d_a, f, (size_t)cells * n * sizeof(double), cudaMemcpyHostToDevice));

  double rho0[64], u0[64 * 3], T0[64], rho[64], u[64 * 3], T[64];
  CHECK(fks_moments(ctx, d_a, d_rho, d_u, d_T));
  CUDA(cudaMemcpy(rho0, d_rho, sizeof(rho0), cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(u0, d_u, sizeof(u0), cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(T0, d_T, sizeof(T0), cudaMemcpyDeviceToHost));
  double worst_rho = 0.0, worst_e = 0.0;
  for (int s = 0; s < steps; ++s) {
    CHECK(fks_step(ctx, d_a, d_b, dt));
    double* t = d_a;
    d_a = d_b;
    d_b = t;
    CHECK(fks_moments(ctx, d_a, d_rho, d_u, d_T));
    CUDA(cudaMemcpy(rho, d_rho, sizeof(rho), cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(u, d_u, sizeof(u), cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(T, d_T, sizeof(T), cudaMemcpyDeviceToHost));
    for (int c = 0; c < cells; ++c) {
      const double e0 = rho0[c] * (3.0 * T0[c] + u2(u0, c));  /* 2 x energy density */
      const double e1 = rho[c] * (3.0 * T[c] + u2(u, c));
      worst_rho = fmax(worst_rho, fabs(rho[c] / rho0[c] - 1.0));
      worst_e = fmax(worst_e, fabs(e1 / e0 - 1.0));
    }
  }
  CHECK(fks_check(ctx));
  const double txx0 = txx(f + (size_t)63 * n, N, L, u0[3 * 63]);
  CUDA(cudaMemcpy(f, d_a, (size_t)cells * n * sizeof(double), cudaMemcpyDeviceToHost));
  const double txx1 = txx(f + (size_t)63 * n, N, L, u[3 * 63]);
  int64_t nstep = 0;
  double dt_run = 0.0;
  CHECK(fks_get_state(ctx, &nstep, &dt_run));
  printf("fks_demo: %d cells of %d^3, %lld steps (dt %.3g), %lld kernel launches\n", cells, N, (long long)nstep,
         dt_run, (long long)fks_launch_count(ctx));
  printf("fks_demo: max relative drift: mass %.2e, energy %.2e; cell 63: T %.6f -> %.6f, T_xx %.6f -> %.6f\n",
         worst_rho, worst_e, T0[63], T[63], txx0, txx1);
  CHECK(fks_finalize(ctx));
  cudaFree(d_a);
  cudaFree(d_b);
  cudaFree(d_rho);
  cudaFree(d_u);
  cudaFree(d_T);
  free(f);
  return (worst_rho < 1e-12 && worst_e < 1e-12 && nstep == steps && fabs(txx1 - T[63]) < fabs(txx0 - T0[63])) ? 0 : 2;
}
