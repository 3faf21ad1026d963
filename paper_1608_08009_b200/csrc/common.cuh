// Shared device-side definitions: kernel parameter blocks and the FKS transport gather.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fks {

#ifndef FKS_KMAXN
#define FKS_KMAXN 64
#endif
constexpr int kMaxN = FKS_KMAXN;  // velocity nodes per axis (N = 64: 2D only)

// Checked build (FKS_CHECKS=1 python -m paper_1608_08009_b200.build -> libfks_checked.so): every
// global / exchange-ring / table / shared-memory / TMEM index the kernels form is range-checked and
// the kernel traps on a violation -- the bounds-and-asserts substitute for compute-sanitizer, which
// this GPU pool does not allow (profiles/r02_sanitizer.txt).  Compiled out otherwise.
#ifdef FKS_CHECKS
#define FKS_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define FKS_CHECK(cond) do { } while (0)
#endif

// a1 + a3: per-step shift table and boundary description.
struct TransportParams {
  int dx;                  // space dimension 0..3
  int M[3];                // local cells per space axis (axis 0 fastest)
  int bc[6];               // FKS_BC_* per face
  int cfl1;                // every |delta| <= 1 (the 3^dx-sources fast paths apply)
  int reflect;             // NEXT-1: specular reflection at solid cells (needs solid)
  int Nv;                  // velocity nodes per axis (mirror index N-1-k)
  const uint8_t* solid;    // [local cells] solid mask (nullptr: none)
  int8_t delta[3][kMaxN];  // delta[a][k_a] = s^{n+1} - s^n for velocity component a
  const double* ghost[6];  // ghost vectors (n values) of GHOST faces, device memory
  const double* halo[2];   // HALO faces of the slowest axis: neighbour rank's boundary plane
                           // [plane cells][n] (cells in C order over the other axes)
  const uint8_t* halo_solid[2];  // solid flags of the neighbour planes (specular reflection on a
                                 // partitioned grid; nullptr: none)
  int64_t ncells_total;    // local cells of the state arrays (checked build)
  int64_t plane_cells;     // cells per plane of the slowest axis (checked build)
};

struct StepParams {
  const double* f_in;        // F^n       [cells][n]
  double* f_out;             // F^{n+1} or Q [cells][n]
  const double2* tables;     // folded tables, layout per kernel (see kernels*.cu)
  double2* scratch;          // per-group exchange buffers (3D)
  unsigned* sync;            // per-group synchronisation counters (3D; zeroed before each launch)
  int* nonfinite;            // device flag
  const int* cell_list;      // fluid cells to process (local linear indices)
  int ncells;                // entries of cell_list
  int A;                     // directions (tables hold A + 1 entries, the last is the loss)
  int mode;                  // 0 = collide (write Q), 1 = step (project + Euler),
                             // 2 = Heun stage: f_out = (f_base + f_in + dt/tau Pi Q(f_in)) / 2 (NEXT-4)
  const double* f_base;      // mode 2: f* of the step [cells][n] (same cell indices as f_in)
  int64_t table_elems;       // double2 entries behind `tables` (checked build)
  int project;               // apply a8
  double dt_tau;             // dt / tau
  double L, dv;              // velocity box half-width and spacing
  double Ginv[25];           // (Phi Phi^T)^{-1}, (dv+2)^2 row-major
  TransportParams tp;
};

// NEXT-2 BGK step (kernels_bgk.cu).
struct BgkParams {
  const double* f_in;
  double* f_out;
  int* nonfinite;
  const int* cell_list;  // fluid cells (nullptr: all)
  int ncells;
  int nu_rule;           // 0: nu = rho, 1: nu = mu, 2: Euler limit (F = E[f*])
  double mu;
  double dt_tau;
  double L, dv;
  double Ginv[25];       // (Phi Phi^T)^{-1}, (dv+2)^2 row-major
  TransportParams tp;
};

// Coordinates of a local cell along each space axis (computed once per cell, not per element).
struct CellCoord {
  int j[3];
  int64_t cell;
};

__device__ __forceinline__ CellCoord cell_coord(const TransportParams& tp, int64_t cell) {
  CellCoord c;
  c.cell = cell;
  int64_t rem = cell;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a < tp.dx) {
      c.j[a] = (int)(rem % tp.M[a]);
      rem /= tp.M[a];
    } else {
      c.j[a] = 0;
    }
  }
  return c;
}

// f*_cell[k]: the transported value for velocity k = (kx, ky, kz) (P:243-257 eq. f_bar sampled
// at x_j).  Out-of-domain sources: PERIODIC wraps, OUTFLOW clamps, GHOST reads the
// face's ghost vector (the lowest axis with a ghost face wins; reading #19).  A HALO
// face (only on the slowest axis) reads the neighbour slab's boundary plane -- the ghost cells
// of the paper's z-slab decomposition (Fig. mpi-decomp).
// delta: the shift table [3][kMaxN] (a shared-memory copy of tp.delta in the hot kernels: its
// index varies across a warp, which serialises constant-bank loads).
// Where f*_cell reads velocity k from when the per-axis shifts of k are d[a] (a < tp.dx): the
// returned base satisfies f*_cell[k] = base[k] -- the source cell's vector, a ghost vector or a
// halo plane (the rules of gather_fstar below).
__device__ __forceinline__ const double* source_base(const double* __restrict__ F, const TransportParams& tp,
                                                     const CellCoord& cc, const int (&d)[3], int n) {
  if (tp.dx == 0) return F + cc.cell * n;
  int64_t src = 0, stride = 1, hplane = 0;
  int gface = -1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a < tp.dx) {
      const int Ma = tp.M[a];
      int s = cc.j[a] + d[a];
      if (s < 0) {
        const int b = tp.bc[2 * a];
        if (b == 0) { s %= Ma; if (s < 0) s += Ma; }  // true modulo: |d| may exceed M_a (CFL > 1)
        else { if ((b == 1 || b == 3) && gface < 0) { gface = 2 * a; hplane = src; } s = 0; }
      } else if (s >= Ma) {
        const int b = tp.bc[2 * a + 1];
        if (b == 0) s %= Ma;
        else { if ((b == 1 || b == 3) && gface < 0) { gface = 2 * a + 1; hplane = src; } s = Ma - 1; }
      }
      src += s * stride;
      stride *= Ma;
    }
  }
  if (gface >= 0) {
    if (tp.bc[gface] == 3) {
      FKS_CHECK(tp.halo[gface & 1] != nullptr && hplane >= 0 && hplane < tp.plane_cells);
      return tp.halo[gface & 1] + hplane * n;
    }
    FKS_CHECK(tp.ghost[gface] != nullptr);
    return tp.ghost[gface];
  }
  FKS_CHECK(src >= 0 && src < tp.ncells_total);
  return F + src * n;
}

// NEXT-1 (specular reflection, oracle/transport.gather_specular): undo the per-axis moves in
// reverse axis order from cell j; a move whose origin is an in-domain solid cell was a reflection
// instead (component a mirrored, no move).  Returns the source of the remaining shifts (face rules
// of source_base) and the mask of mirrored velocity components.
__device__ __forceinline__ const double* source_resolve(const double* __restrict__ F, const TransportParams& tp,
                                                        const CellCoord& cc, int (&d)[3], int n, int& flip) {
  flip = 0;
  if (tp.reflect) {
    int c[3] = {cc.j[0], cc.j[1], cc.j[2]};
#pragma unroll
    for (int a = 2; a >= 0; --a) {
      if (a >= tp.dx || d[a] == 0) continue;
      int nb = c[a] + d[a];
      if (tp.bc[d[a] < 0 ? 2 * a : 2 * a + 1] == 0) {  // PERIODIC: true modulo (|d| may exceed M_a)
        nb %= tp.M[a];
        if (nb < 0) nb += tp.M[a];
      }
      // the candidate origin is a solid cell only if EVERY coordinate is inside the domain (an
      // axis undone earlier may have left c[b] outside through an OUTFLOW / GHOST / HALO face) --
      // or, on a partitioned grid, inside the neighbour plane of a HALO face of the slab axis
      // (solid flags exchanged with the planes, tp.halo_solid)
      const int sa = tp.dx - 1;
      int hs = -1;  // HALO face whose neighbour plane holds the candidate
      bool inside = true;
      int64_t idx = 0, stride = 1;
      for (int b = 0; b < tp.dx; ++b) {
        const int cb = b == a ? nb : c[b];
        if (cb < 0 || cb >= tp.M[b]) {
          const int face = cb < 0 ? 2 * b : 2 * b + 1;
          if (b == sa && tp.bc[face] == 3 && (cb == -1 || cb == tp.M[b]) && tp.halo_solid[face & 1]) hs = face & 1;
          else inside = false;
        } else if (b < sa) {
          idx += (int64_t)cb * stride;
          stride *= tp.M[b];
        } else {
          idx += (int64_t)cb * stride;
        }
      }
      bool is_solid = false;
      if (inside) {
        if (hs >= 0) {
          FKS_CHECK(idx >= 0 && idx < tp.plane_cells);
          is_solid = tp.halo_solid[hs][idx] != 0;
        } else {
          FKS_CHECK(idx >= 0 && idx < tp.ncells_total);
          is_solid = tp.solid[idx] != 0;
        }
      }
      if (is_solid) {
        flip |= 1 << a;
        d[a] = 0;
      } else {
        c[a] = nb;
      }
    }
  }
  return source_base(F, tp, cc, d, n);
}

// velocity index k with the components in `flip` mirrored (k_a -> N-1-k_a)
__device__ __forceinline__ int mirror_k(int k, int kx, int ky, int kz, int flip, int N) {
  if (flip & 1) k += N - 1 - 2 * kx;
  if (flip & 2) k += (N - 1 - 2 * ky) * N;
  if (flip & 4) k += (N - 1 - 2 * kz) * N * N;
  return k;
}

__device__ __forceinline__ double gather_fstar(const double* __restrict__ F, const TransportParams& tp,
                                               const CellCoord& cc, int k, int kx, int ky, int kz, int n,
                                               const int8_t (*delta)[kMaxN]) {
  FKS_CHECK(k >= 0 && k < n && cc.cell >= 0 && cc.cell < tp.ncells_total);
  if (tp.dx == 0) return F[cc.cell * n + k];
  int d[3] = {delta[0][kx], tp.dx > 1 ? delta[1][ky] : 0, tp.dx > 2 ? delta[2][kz] : 0};
  if (tp.reflect) {
    int flip;
    const double* base = source_resolve(F, tp, cc, d, n, flip);
    const int km = mirror_k(k, kx, ky, kz, flip, tp.Nv);
    FKS_CHECK(km >= 0 && km < n);
    return base[km];
  }
  return source_base(F, tp, cc, d, n)[k];
}

// Copy the shift table into shared memory (call with all threads, then __syncthreads()).
__device__ __forceinline__ void load_delta(const TransportParams& tp, int8_t (*sdelta)[kMaxN]) {
  for (int i = threadIdx.x; i < 3 * kMaxN; i += blockDim.x) sdelta[i / kMaxN][i % kMaxN] = tp.delta[i / kMaxN][i % kMaxN];
}

__device__ __forceinline__ double node_v(int k, double L, double dv) { return -L + (k + 0.5) * dv; }

}  // namespace fks
