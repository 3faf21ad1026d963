// Launchers of the device kernels (host-callable, used by fks_api.cu).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace fks {

// 3D (hard spheres): a group of 8 co-resident CTAs per cell (cooperative launch, one CTA per
// SM); scratch = ngroups * scratch_elems3d(N) double2, sync = ngroups * sync_bytes3d() bytes,
// zeroed before every launch.
cudaError_t launch_step3d(int N, const StepParams& p, int ngroups, cudaStream_t s);
int max_active_clusters3d(int N);  // groups that fit the GPU at once
size_t scratch_elems3d(int N);
size_t sync_bytes3d();
// 3D table layout: P CTAs per cell, NP l_y planes per CTA, slabr rows (of N entries) per CTA slab.
int table_layout3d(int N, int* P, int* NP, int* slabr);

// 3D, N = 64 (kernels3d64.cu): a group of 64 co-resident CTAs per cell (cooperative launch, two
// CTAs per SM); scratch = ngroups * scratch_elems3d64() double2, sync = ngroups * sync_bytes3d64()
// bytes, zeroed before every launch.  Tables in the full layout T[p][n].
cudaError_t launch_step3d64(const StepParams& p, int ngroups, cudaStream_t s);
int max_groups3d64();
size_t scratch_elems3d64();
size_t sync_bytes3d64();

// N = 4 (kernels_small.cu), 2D and 3D: one thread per velocity point, transforms in SMEM.
cudaError_t launch_step_small(int N, int dv, const StepParams& p, int sm_count, cudaStream_t s);

// 2D with pencils split over lane pairs (kernels2dp.cu): N = 64 (2 cells per 256-thread CTA) and
// N = 32 (8 cells per 512-thread CTA, tables in SMEM when (A + 1) directions fit).
cudaError_t launch_step2d_pair(int N, const StepParams& p, int nblocks, cudaStream_t s);
int cells_per_block2d_pair(int N);
bool step2d_pair_fits(int N, int A);
// Which 2D kernel runs for (N, A): the pair kernel for N = 64 always, for N = 32 when it fits and
// FKS_2D_PAIR (development knob) does not say otherwise.
bool use_pair2d(int N, int A);

// 2D (Maxwell molecules): cells_per_block2d(N) cells per CTA.
cudaError_t launch_step2d(int N, const StepParams& p, int nblocks, cudaStream_t s);
int cells_per_block2d(int N);

// a1 + a3 only: f_out[c] = f*[c] for all local cells (solid cells copied unchanged).
cudaError_t launch_transport(const double* f_in, double* f_out, const TransportParams& tp, const uint8_t* solid,
                             int64_t ncells, int n, int N, int dv, cudaStream_t s);

// a2: velocity slices exchanged with a neighbour slab (k along the slab axis).
struct SliceList {
  int n;
  int8_t k[kMaxN];
};
// pack: buf = f[first_cell .. first_cell + pc)[slices]; unpack: f[...][slices] = buf.
cudaError_t launch_halo_pack(const double* f, int64_t first_cell, int pc, int n, int N, int dv, int axis,
                             const SliceList& sl, double* buf, bool unpack, cudaStream_t s);

// Copy the listed cells f_out[c] = f_in[c] (solid cells in fks_step).
cudaError_t launch_copy_cells(const double* f_in, double* f_out, const int* cells, int count, int n, cudaStream_t s);

// NEXT-2: BGK relaxation step (transport gather + conservative Maxwellian + forward Euler).
cudaError_t launch_bgk(int N, int dv, const BgkParams& p, int sm_count, cudaStream_t s);

// a10: rho, u[dv], T per cell.
cudaError_t launch_moments(const double* f, double* rho, double* u, double* T, int64_t ncells, int N, int dv,
                           double L, double dv_spacing, cudaStream_t s);

}  // namespace fks
