/*
 * fks.h -- C ABI of libfks, the B200-native hot path of the FKS + fast-spectral Boltzmann
 * solver of Dimarco, Loubere, Narski and Rey (arXiv 1608.08009).
 *
 * Citation keys: P:n = PAPER.md line n (section / equation named beside it).
 *
 * What the library computes, per physical cell j and velocity node k:
 *   a1  shift table     delta_k = s^{n+1}_k - s^n_k, s^n_k = floor(1/2 - n (v_k dt)/dx)
 *                       (P:243-253 eq. f_bar; P:560-561 eq. transport)
 *   a3  transport       f*_j[k] = F^n[j + delta_k][k] with periodic / ghost / outflow faces
 *                       (sampling at x_j P:269-271)
 *   a4-a7 collision     Q(f*) = fast spectral Carleman quadrature with A directions
 *                       (P:390-452 eq. ode/FKM, 2D tables, 3D tables)
 *   a8  projection      Pi Q = Q - Phi^T (Phi Phi^T)^{-1} Phi Q (P:319-358 eq. minim1)
 *   a9  Euler           F^{n+1}_j = f*_j + (dt/tau) Pi Q_j  (P:273-275 eq. f_coll)
 *   a10 moments         rho, u, T
 *
 * Conventions.
 *  - Velocity lattice: N points per axis on [-L, L), cell-centred nodes
 *    v_k = -L + (k + 1/2) 2L/N (reading #14).  n = N^dv.
 *  - Layout of every distribution array: f[local_cell][k], fp64, k in C order over velocity
 *    axes with v_x fastest (k = kx + N*ky + N*N*kz); cells in C order over the local grid
 *    with space axis 0 fastest.
 *  - Array pointers are DEVICE pointers owned by the caller unless the name says _host.
 *    All device work is enqueued on the context stream (fks_set_stream; default stream 0)
 *    and is asynchronous unless stated otherwise.  The library never frees caller memory.
 *  - Errors: argument errors return FKS_E_INVAL / FKS_E_UNSUPPORTED synchronously with
 *    nothing enqueued; CUDA launch/API failures return FKS_E_CUDA; a non-finite value
 *    produced by fks_step sets a device flag that fks_check() reports as FKS_E_NONFINITE.
 *    There is no CPU fallback: without a usable sm_100 device fks_init returns FKS_E_CUDA.
 *  - A context is not thread-safe; use one per (process, device).
 */
#ifndef FKS_H
#define FKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fks_ctx fks_ctx;
typedef struct fks_loopback fks_loopback;  /* in-process communicator (tests on one device) */

typedef enum {
  FKS_OK = 0,
  FKS_E_INVAL = -1,
  FKS_E_UNSUPPORTED = -2,
  FKS_E_NOMEM = -3,
  FKS_E_CUDA = -4,
  FKS_E_NCCL = -5,
  FKS_E_NONFINITE = -6,
  FKS_E_STATE = -7
} fks_status;

/* Face kinds (reading #19).  FKS_BC_HALO marks a face of the slowest space axis that
 * borders another rank's slab (the paper's MPI z-slab ghost cells); its sources are
 * read from the plane set with fks_set_halo. */
enum { FKS_BC_PERIODIC = 0, FKS_BC_GHOST = 1, FKS_BC_OUTFLOW = 2, FKS_BC_HALO = 3 };

typedef struct {
  int dv;          /* velocity dimension: 2 (Maxwell molecules) or 3 (hard spheres)          */
  int dx;          /* space dimension 0..3; 0 = a batch of independent homogeneous cells    */
  int64_t M[3];    /* local cells per space axis (axis 0 fastest); dx = 0: M[0] = batch size */
  double h;        /* Delta x, equal on all axes                                    */
  int bc[6];       /* face kinds [lo0, hi0, lo1, hi1, lo2, hi2] (ignored when dx = 0)       */
} fks_grid;

/* Create a context (P:85-91 model; P:141-158 kernels).
 *   grid          physical grid (copied).
 *   Nv            points per velocity axis: 4, 8, 16, 32 or 64 (4 <= N <= 64, S:28;
 *                 the paper uses 8..64 per axis); else FKS_E_INVAL.
 *   L             velocity box half-width (> 0).
 *   M_dirs        number of quadrature directions A: dv = 2 -> theta_p = pi p / A, p = 1..A
 *                 (P:490); dv = 3 -> 24 = the spherical 7-design (reading #17), a perfect
 *                 square A1^2 = the (theta, phi) product grid of P:527-540 (reading #6);
 *                 anything else needs fks_set_dirs.
 *   kernel_gamma  VHS exponent gamma of B = C |q|^gamma (the paper's alpha), -1 < gamma <= 2,
 *                 else FKS_E_UNSUPPORTED.  gamma = dv - 2 (2D Maxwell molecules, 3D hard spheres)
 *                 makes Btilde constant and the tables closed forms;
 *                 any other gamma uses the decoupled model Btilde(x, y) = 2^{dv-1} C |x|^{gamma-(dv-2)},
 *                 b = 1 (NEXT-3, reading #25): alpha_p = phi_{R,a}(l . e_p) with
 *                 phi_{R,a}(s) = int_{-R}^{R} |rho|^gamma e^{i rho s} d rho by 160-point Gauss-Jacobi
 *                 quadrature, alpha'_p unchanged; the kernels are the same.
 * Defaults: tau = 1, b0 = 1/(2 pi) (2D) or C1 = 1/(4 pi) (3D) (reading #7), R = 2 lambda pi
 * (reading #1), projection on.  Builds the fp64 tables on the host and uploads them.
 * Returns FKS_E_CUDA if no sm_100 device is present. */
fks_status fks_init(const fks_grid* grid, int Nv, double L, int M_dirs, double kernel_gamma, fks_ctx** out);

/* tau, kernel constant b0 / C1 (<= 0 keeps the default), scaled truncation radius R
 * (<= 0 keeps the default), project (0/1).  Rebuilds the tables. */
fks_status fks_set_params(fks_ctx* ctx, double tau, double kernel_const, double R, int project);

/* Replace the direction set: e_host [M][dv] unit vectors, w_host [M] weights (host memory,
 * copied).  For dv = 2 the perpendicular partner of e is e rotated by +pi/2. */
fks_status fks_set_dirs(fks_ctx* ctx, const double* e_host, const double* w_host, int M);

/* Ghost vector for a GHOST face (n values, device memory, copied into library memory). */
fks_status fks_set_ghost(fks_ctx* ctx, int face, const double* ghost_f);

/* Neighbour planes for the FKS_BC_HALO faces (a2, the slab exchange): lo_plane / hi_plane are
 * device pointers to [plane cells][n] (the plane just below / above the local slab along the
 * slowest axis, cells in C order over the other axes).  The pointers are used by the next
 * fks_step / fks_transport calls (not copied); NULL for a face without a HALO. */
fks_status fks_set_halo(fks_ctx* ctx, const double* lo_plane, const double* hi_plane);

/* a2 fused into the step over peer memory: a rank maps its neighbours' state buffers (CUDA IPC;
 * NVLink / NVSwitch peers of one box, or another process on the same GPU) and hands fks_set_halo
 * pointers to THEIR boundary planes -- the lower neighbour's last plane, the upper one's first --
 * so the step's transport gather reads the sources across the slab face straight from the peer:
 * no pack, send, receive or unpack (paper_1608_08009_b200.parallel.PeerHalo).  The
 * caller orders the ranks' steps (a stream-ordered barrier per step: a rank's step n + 1 reads the
 * neighbours' step-n output, and their step n + 2 overwrites the buffer it read).  Specular walls
 * across the face need the neighbours' solid flags: library exchange only (fks_set_comm).
 *   fks_ipc_get_handle: handle_out (FKS_IPC_HANDLE_BYTES bytes) of the device allocation that
 *                       contains dptr, and the byte offset of dptr inside it;
 *   fks_ipc_open:       maps a handle from another process; *base_out = the allocation base
 *                       (add the owner's offset); FKS_E_CUDA if the peer cannot be mapped;
 *   fks_ipc_close:      unmaps it. */
#define FKS_IPC_HANDLE_BYTES 64
fks_status fks_ipc_get_handle(const void* dptr, void* handle_out, int64_t* offset_out);
fks_status fks_ipc_open(const void* handle, void** base_out);
fks_status fks_ipc_close(void* base);

/* a2 inside the library: the slab halo exchange of the paper's MPI z-slab decomposition
 * (Fig. mpi-decomp; ghost cells exchanged every step) over NCCL (NVLink /
 * NVSwitch between the GPUs of a box), one rank per GPU.  The slab axis is the slowest space axis
 * (dx - 1); its HALO faces name the neighbours: lo face -> rank - 1, hi face -> rank + 1 (mod nranks,
 * so a periodic global axis is a ring).  Per step only the velocity slices whose FKS shift crosses
 * the face are sent (k_a with delta = +1 to the lower rank, -1 to the upper one; halo width 1 at
 * CFL <= 1), packed on a library communication stream, exchanged with grouped ncclSend/ncclRecv and
 * unpacked into library-owned neighbour planes; fks_step runs the interior cells while the exchange
 * is in flight and the cells of the HALO-face planes after it.  fks_transport and fks_step_bgk use
 * the same exchange (before their kernel).  A comm replaces fks_set_halo.
 *
 * fks_comm_unique_id: a new NCCL unique id (128 bytes) -- call on one rank, broadcast the bytes
 *   (e.g. torch.distributed), then every rank calls fks_set_comm with it.  NCCL is loaded at run
 *   time (dlopen libnccl.so.2, reusing an already loaded copy); FKS_E_NCCL if unavailable or an
 *   NCCL call fails.
 * fks_set_comm: build this rank's communicator (collective over the nranks processes).  dx >= 1;
 *   once per context.  With specular reflection (fks_set_specular) the boundary planes' solid
 *   flags travel with the planes, so walls that straddle a slab face reflect as in one domain.
 * fks_comm_loopback_create / fks_set_comm_loopback: the same exchange between contexts of ONE
 *   process through device copies (all ranks on one GPU, driven in turn): every rank must call
 *   fks_halo_post for the step before any rank steps (FKS_E_STATE otherwise).
 * fks_halo_post: pack and send this step's planes of f_in now (optional with NCCL: fks_step posts
 *   for itself); dt must already be fixed (a first step or fks_set_state), else FKS_E_STATE.
 * fks_get_comm_stats: payload bytes sent by the last exchange (both faces), and the fluid cells run
 *   before / after the exchange completes. */
fks_status fks_comm_unique_id(void* nccl_unique_id_out);
fks_status fks_set_comm(fks_ctx* ctx, const void* nccl_unique_id, int rank, int nranks);
fks_status fks_comm_loopback_create(int nranks, fks_loopback** out);
fks_status fks_comm_loopback_destroy(fks_loopback* loop);
fks_status fks_set_comm_loopback(fks_ctx* ctx, fks_loopback* loop, int rank);
fks_status fks_halo_post(fks_ctx* ctx, const double* f_in);
fks_status fks_get_comm_stats(const fks_ctx* ctx, int64_t* bytes_sent_last, int* interior_cells, int* boundary_cells);

/* Solid mask (host, one byte per local cell, copied): solid cells are not collided and keep
 * their values (reading #19; fks_set_specular reflects at them instead). NULL clears it. */
fks_status fks_set_solid(fks_ctx* ctx, const uint8_t* solid_host);

/* NEXT-1: specular reflection at solid cells instead of the frozen solid values of reading #19
 * ("reflective boundary conditions"; reading #23): in the transport gather of
 * fks_transport / fks_step / fks_step_bgk, a particle whose per-axis move would end in a solid
 * cell is reflected there (velocity component mirrored, k_a -> N-1-k_a) -- the inverse of the
 * forward bounce map, so a closed box conserves mass and energy exactly.  on = 0 restores the
 * default.  On a partitioned grid (HALO faces) the neighbours' solid flags come with the library
 * exchange (fks_set_comm / fks_set_comm_loopback); with caller-owned halo planes (fks_set_halo)
 * the steps return FKS_E_UNSUPPORTED. */
fks_status fks_set_specular(fks_ctx* ctx, int on);

/* NEXT-4 (reading #26): the time scheme of fks_step.
 *   splitting  FKS_SPLIT_LIE (default; transport then collision) or FKS_SPLIT_STRANG
 *              ("high order time splitting": f^{n+1} = T(dt/2) C(dt) T(dt/2) f^n, the
 *              half transports being FKS gathers between the half-step positions 2n -> 2n+1 -> 2n+2,
 *              s = floor(1/2 - (p c) / 2); identical to Lie without spatial axes).
 *   integrator FKS_TIME_EULER (default; eq. f_coll) or FKS_TIME_HEUN ("many
 *              different time integrators can be employed": explicit RK2, f1 = f* + dt/tau PiQ(f*),
 *              f^{n+1} = (f* + f1 + dt/tau PiQ(f1)) / 2 -- two collision passes per step).
 * Non-default schemes use one library-owned state-sized scratch buffer (allocated on first use).
 * FKS_E_UNSUPPORTED for Strang on a partitioned grid (HALO faces: the second half transport would
 * need a second exchange); fks_step_bgk supports Strang but not Heun (FKS_E_UNSUPPORTED). */
enum { FKS_SPLIT_LIE = 0, FKS_SPLIT_STRANG = 1 };
enum { FKS_TIME_EULER = 0, FKS_TIME_HEUN = 1 };
fks_status fks_set_scheme(fks_ctx* ctx, int splitting, int integrator);

/* Stream (a cudaStream_t passed as void*) on which all later work is enqueued. */
fks_status fks_set_stream(fks_ctx* ctx, void* cuda_stream);

/* a4-a7: Q[cell][k] = Q(f[cell]) for every local cell, unprojected, user units, no 1/tau.
 * In-place calls: here and in fks_transport / fks_step / fks_step_bgk the output
 * may be the input pointer itself -- the result then goes to a library-owned state-sized buffer
 * (allocated on first use) and one device-to-device copy on the context stream moves it back.
 * Partially overlapping buffers are invalid (not detected). */
fks_status fks_collide(fks_ctx* ctx, const double* f, double* Q);

/* a1 + a3: f_out = transported f_in for the step n -> n+1, then n += 1 (collision skipped).
 * dt must equal the context dt once one was set (it is fixed per run, reading #15). */
fks_status fks_transport(fks_ctx* ctx, const double* f_in, double* f_out, double dt);

/* a1..a9 fused: f_out = F^{n+1} from f_in = F^n, then n += 1 (f_out == f_in: in place, see
 * fks_collide).  One launch (plus a solid-cell copy when the grid has solids) with the default
 * scheme; see fks_set_scheme. */
fks_status fks_step(fks_ctx* ctx, const double* f_in, double* f_out, double dt);

/* fks_step with HOST buffers: copies f_in_host to the device, steps, copies the result back
 * to f_out_host and synchronises (end-to-end path; pinned memory recommended).  The batch is
 * processed in chunks so that the host->device copy, the step and the device->host copy of
 * consecutive chunks overlap (two library-owned copy streams): cells for dx = 0 without solids,
 * planes of the slowest axis for dx > 0 (a chunk steps once the next chunk's first plane landed;
 * not with a periodic or HALO slab axis, a comm, CFL > 1 along it, or a non-default scheme, which
 * take the one-shot path).  The result is bitwise that of fks_step. */
fks_status fks_step_host(fks_ctx* ctx, const double* f_in_host, double* f_out_host, double dt);

/* NEXT-2 (beyond the Boltzmann hot path): one BGK step, F = f* + (dt/tau) nu (E[f*] - f*), with
 * the transport gather of fks_step (a1+a3) and the conservative Maxwellian E of eq. minimMax
 * (the Maxwellian of the cell's moments projected onto them, so mass, momentum and
 * energy are exact).  nu_rule: FKS_NU_RHO (nu = rho), FKS_NU_CONST (nu = mu > 0),
 * FKS_NU_EULER (the tau -> 0 limit, F = E[f*]).  tau from fks_set_params.  Advances the step
 * counter like fks_step; solid cells are copied.  Device pointers (f_out == f_in: in place). */
enum { FKS_NU_RHO = 0, FKS_NU_CONST = 1, FKS_NU_EULER = 2 };
fks_status fks_step_bgk(fks_ctx* ctx, const double* f_in, double* f_out, double dt, int nu_rule, double mu);

/* a10: rho[cell], u[cell][dv], T[cell] (T = int |v-u|^2 f / (dv rho), reading #12). */
fks_status fks_moments(fks_ctx* ctx, const double* f, double* rho, double* u, double* T);

/* Step counter n and time step dt (checkpoint / resume: shifts are pure functions of n). */
fks_status fks_get_state(fks_ctx* ctx, int64_t* n, double* dt);
fks_status fks_set_state(fks_ctx* ctx, int64_t n, double dt);

/* Synchronise the stream; FKS_E_NONFINITE if any step produced a non-finite value since
 * the last check (the flag is then cleared), FKS_E_CUDA on an asynchronous CUDA error. */
fks_status fks_check(fks_ctx* ctx);

/* Number of kernel launches the library has enqueued since the context was created. */
int64_t fks_launch_count(const fks_ctx* ctx);

fks_status fks_finalize(fks_ctx* ctx);
const char* fks_strerror(fks_status s);

/* ---- host-only introspection (no device needed; used by the CPU tests) ---------------- */

/* The spectral tables exactly as uploaded, before folding (reading #10):
 * alpha_host, alphap_host: [A][n] in FFT mode order (same layout as f), D_host: [n],
 * w_host: [A], e_host: [A][dv].  Arrays may be NULL.  Returns the node-space factor
 * s = Btilde kappa^{-(dv+gamma)} in *scale.  Arguments as in fks_init / fks_set_params. */
fks_status fks_host_tables(int dv, int Nv, double L, int M_dirs, double R, double kernel_const,
                           double kernel_gamma, double* alpha_host, double* alphap_host, double* D_host,
                           double* w_host, double* e_host, double* scale);

/* a2 plan of step n: the velocity indices k (along the slab axis) whose slices the exchange sends to
 * the lower rank (delta = +1) and to the upper rank (delta = -1); arrays of Nv entries.
 * FKS_E_UNSUPPORTED if some |delta| > 1 (halo width 1). */
fks_status fks_host_halo_slices(int64_t n, int Nv, double L, double dt, double h, int8_t* to_lower, int* n_lower,
                                int8_t* to_upper, int* n_upper);

/* delta_k = s^{n+1}_k - s^n_k for the N nodes of one velocity axis (a1). */
fks_status fks_host_shift(int64_t n, int Nv, double L, double dt, double h, int8_t* delta_host);

#ifdef __cplusplus
}
#endif
#endif /* FKS_H */
