"""Thin Python binding of the libfks C ABI (include/fks.h): same names, argument marshalling only.

Device arrays are torch float64 CUDA tensors (plumbing: device memory and streams); every
step of the hot path runs in the library's kernels.  No function here computes any part of
the method, and nothing falls back to the CPU.
"""
import ctypes

import numpy as np

from ._lib import FksError, FksGrid, check, load  # noqa: F401

BC_PERIODIC, BC_GHOST, BC_OUTFLOW, BC_HALO = 0, 1, 2, 3
NU_RHO, NU_CONST, NU_EULER = 0, 1, 2  # fks_step_bgk collision-frequency rules (include/fks.h)
SPLIT_LIE, SPLIT_STRANG = 0, 1         # fks_set_scheme (NEXT-4)
TIME_EULER, TIME_HEUN = 0, 1


def _ptr(t):
    """Device pointer of a contiguous float64 CUDA tensor."""
    if not (t.is_cuda and t.dtype.is_floating_point and t.element_size() == 8 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Context:
    """Owns one fks_ctx* (fks_init ... fks_finalize)."""

    def __init__(self, dv, dx, M, Nv, L, M_dirs, kernel_gamma=None, h=1.0, bc=None):
        lib = load()
        g = FksGrid()
        g.dv, g.dx = dv, dx
        Ms = list(M) + [1] * (3 - len(M))
        for a in range(3):
            g.M[a] = int(Ms[a])
        g.h = float(h)
        bc = list(bc or []) + [0] * (6 - len(bc or []))
        for f in range(6):
            g.bc[f] = int(bc[f])
        if kernel_gamma is None:
            kernel_gamma = 0.0 if dv == 2 else 1.0
        h_ = ctypes.c_void_p()
        check(lib.fks_init(ctypes.byref(g), Nv, float(L), M_dirs, float(kernel_gamma), ctypes.byref(h_)), "fks_init")
        self._lib, self.handle = lib, h_
        self.dv, self.dx, self.N, self.L = dv, dx, Nv, L
        self.n = Nv ** dv
        self.ncells = int(np.prod([int(m) for m in (M if dx else M[:1])]))

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.fks_finalize(self.handle)
            self.handle = None

    # ---- configuration -------------------------------------------------------------------
    def set_params(self, tau=1.0, kernel_const=0.0, R=0.0, project=True):
        check(self._lib.fks_set_params(self.handle, float(tau), float(kernel_const), float(R), int(project)),
              "fks_set_params")

    def set_dirs(self, e, w):
        e = np.ascontiguousarray(e, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        check(self._lib.fks_set_dirs(self.handle, _dptr(e), _dptr(w), len(w)), "fks_set_dirs")

    def set_ghost(self, face, ghost):
        check(self._lib.fks_set_ghost(self.handle, face, _ptr(ghost)), "fks_set_ghost")

    def set_halo(self, lo, hi):
        """Neighbour planes (float64 CUDA tensors [plane cells, n]) for the HALO faces, or None."""
        check(self._lib.fks_set_halo(self.handle, _ptr(lo) if lo is not None else None,
                                     _ptr(hi) if hi is not None else None), "fks_set_halo")
        self._halo_refs = (lo, hi)  # keep the buffers alive while the library holds the pointers

    def set_halo_ptr(self, lo, hi):
        """fks_set_halo with raw device addresses (ints, or None): e.g. a peer's boundary plane
        mapped with ipc_open (parallel.PeerHalo).  The caller keeps the memory alive."""
        check(self._lib.fks_set_halo(self.handle, ctypes.c_void_p(lo) if lo is not None else None,
                                     ctypes.c_void_p(hi) if hi is not None else None), "fks_set_halo")
        self._halo_refs = None

    def set_solid(self, mask):
        if mask is None:
            check(self._lib.fks_set_solid(self.handle, None), "fks_set_solid")
            return
        m = np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        check(self._lib.fks_set_solid(self.handle, m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "fks_set_solid")

    def set_specular(self, on=True):
        """NEXT-1: specular reflection at solid cells (fks_set_specular)."""
        check(self._lib.fks_set_specular(self.handle, int(bool(on))), "fks_set_specular")

    def set_scheme(self, splitting=SPLIT_LIE, integrator=TIME_EULER):
        """NEXT-4: splitting SPLIT_LIE / SPLIT_STRANG, integrator TIME_EULER / TIME_HEUN (fks_set_scheme)."""
        check(self._lib.fks_set_scheme(self.handle, int(splitting), int(integrator)), "fks_set_scheme")

    # ---- a2: the slab exchange inside the library -----------------------------------------
    def set_comm(self, unique_id, rank, nranks):
        """fks_set_comm with a 128-byte NCCL unique id (bytes) from comm_unique_id() on one rank."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        check(self._lib.fks_set_comm(self.handle, buf, int(rank), int(nranks)), "fks_set_comm")

    def set_comm_loopback(self, loop, rank):
        """fks_set_comm_loopback: join an in-process Loopback group as `rank`."""
        check(self._lib.fks_set_comm_loopback(self.handle, loop.handle, int(rank)), "fks_set_comm_loopback")
        self._loop_ref = loop

    def halo_post(self, f_in):
        check(self._lib.fks_halo_post(self.handle, _ptr(f_in)), "fks_halo_post")

    def comm_stats(self):
        """(bytes sent by the last exchange, interior fluid cells, boundary fluid cells)."""
        b, i, o = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
        check(self._lib.fks_get_comm_stats(self.handle, ctypes.byref(b), ctypes.byref(i), ctypes.byref(o)),
              "fks_get_comm_stats")
        return b.value, i.value, o.value

    def set_stream(self, stream):
        """stream: a torch.cuda.Stream (or None for the default stream)."""
        check(self._lib.fks_set_stream(self.handle, ctypes.c_void_p(stream.cuda_stream if stream else 0)),
              "fks_set_stream")

    # ---- hot path ------------------------------------------------------------------------
    def collide(self, f, Q):
        check(self._lib.fks_collide(self.handle, _ptr(f), _ptr(Q)), "fks_collide")

    def transport(self, f_in, f_out, dt):
        check(self._lib.fks_transport(self.handle, _ptr(f_in), _ptr(f_out), float(dt)), "fks_transport")

    def step(self, f_in, f_out, dt):
        check(self._lib.fks_step(self.handle, _ptr(f_in), _ptr(f_out), float(dt)), "fks_step")

    def step_bgk(self, f_in, f_out, dt, nu_rule=0, mu=0.0):
        """NEXT-2: one BGK step (fks_step_bgk); nu_rule NU_RHO / NU_CONST (mu) / NU_EULER."""
        check(self._lib.fks_step_bgk(self.handle, _ptr(f_in), _ptr(f_out), float(dt), int(nu_rule), float(mu)),
              "fks_step_bgk")

    def step_host(self, f_in, f_out, dt):
        """f_in, f_out: host float64 arrays/tensors (pinned recommended); synchronous."""
        pi = ctypes.c_void_p(f_in.data_ptr() if hasattr(f_in, "data_ptr") else f_in.ctypes.data)
        po = ctypes.c_void_p(f_out.data_ptr() if hasattr(f_out, "data_ptr") else f_out.ctypes.data)
        check(self._lib.fks_step_host(self.handle, pi, po, float(dt)), "fks_step_host")

    def moments(self, f, rho, u, T):
        check(self._lib.fks_moments(self.handle, _ptr(f), _ptr(rho), _ptr(u), _ptr(T)), "fks_moments")

    # ---- state ---------------------------------------------------------------------------
    def get_state(self):
        n, dt = ctypes.c_int64(), ctypes.c_double()
        check(self._lib.fks_get_state(self.handle, ctypes.byref(n), ctypes.byref(dt)), "fks_get_state")
        return n.value, dt.value

    def set_state(self, n, dt):
        check(self._lib.fks_set_state(self.handle, int(n), float(dt)), "fks_set_state")

    def check(self):
        check(self._lib.fks_check(self.handle), "fks_check")

    def launch_count(self):
        return int(self._lib.fks_launch_count(self.handle))


class Loopback:
    """fks_comm_loopback_create: an in-process communicator for `nranks` contexts on one device."""

    def __init__(self, nranks):
        self._lib = load()
        h = ctypes.c_void_p()
        check(self._lib.fks_comm_loopback_create(int(nranks), ctypes.byref(h)), "fks_comm_loopback_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.fks_comm_loopback_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()


def comm_unique_id():
    """fks_comm_unique_id: 128 bytes to broadcast to every rank before fks_set_comm."""
    buf = ctypes.create_string_buffer(128)
    check(load().fks_comm_unique_id(buf), "fks_comm_unique_id")
    return buf.raw


def ipc_handle(tensor):
    """fks_ipc_get_handle: (64-byte handle, byte offset) of the allocation holding a CUDA tensor."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    check(load().fks_ipc_get_handle(ctypes.c_void_p(tensor.data_ptr()), buf, ctypes.byref(off)),
          "fks_ipc_get_handle")
    return buf.raw, off.value


def ipc_open(handle):
    """fks_ipc_open: map another process's allocation; returns its base address (int)."""
    base = ctypes.c_void_p()
    check(load().fks_ipc_open(ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(base)), "fks_ipc_open")
    return base.value


def ipc_close(base):
    check(load().fks_ipc_close(ctypes.c_void_p(base)), "fks_ipc_close")


# ---- function-style aliases with the C names ---------------------------------------------
def fks_init(dv, dx, M, Nv, L, M_dirs, kernel_gamma=None, h=1.0, bc=None):
    return Context(dv, dx, M, Nv, L, M_dirs, kernel_gamma, h, bc)


def fks_collide(ctx, f, Q):
    ctx.collide(f, Q)


def fks_transport(ctx, f_in, f_out, dt):
    ctx.transport(f_in, f_out, dt)


def fks_step(ctx, f_in, f_out, dt):
    ctx.step(f_in, f_out, dt)


def fks_moments(ctx, f, rho, u, T):
    ctx.moments(f, rho, u, T)


def fks_finalize(ctx):
    ctx.close()


def host_tables(dv, Nv, L, M_dirs, R=0.0, kernel_const=0.0, kernel_gamma=None):
    """fks_host_tables: (alpha [A, n], alphap [A, n], D [n], w [A], e [A, dv], scale)."""
    lib = load()
    if kernel_gamma is None:
        kernel_gamma = 0.0 if dv == 2 else 1.0
    A = M_dirs
    n = Nv ** dv
    al, alp = np.zeros((A, n)), np.zeros((A, n))
    D, w, e = np.zeros(n), np.zeros(A), np.zeros((A, dv))
    s = ctypes.c_double()
    check(lib.fks_host_tables(dv, Nv, float(L), M_dirs, float(R), float(kernel_const), float(kernel_gamma),
                              _dptr(al), _dptr(alp),
                              _dptr(D), _dptr(w), _dptr(e), ctypes.byref(s)), "fks_host_tables")
    return al, alp, D, w, e, s.value


def host_shift(n, Nv, L, dt, h):
    """fks_host_shift: delta_k (int8 [Nv])."""
    out = np.zeros(Nv, dtype=np.int8)
    check(load().fks_host_shift(int(n), Nv, float(L), float(dt), float(h),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_int8))), "fks_host_shift")
    return out


def host_halo_slices(n, Nv, L, dt, h):
    """fks_host_halo_slices: (slices sent to the lower rank, slices sent to the upper rank) of step n."""
    lo, hi = np.zeros(Nv, dtype=np.int8), np.zeros(Nv, dtype=np.int8)
    nl, nh = ctypes.c_int(), ctypes.c_int()
    p8 = ctypes.POINTER(ctypes.c_int8)
    check(load().fks_host_halo_slices(int(n), Nv, float(L), float(dt), float(h), lo.ctypes.data_as(p8), ctypes.byref(nl),
                                      hi.ctypes.data_as(p8), ctypes.byref(nh)), "fks_host_halo_slices")
    return lo[:nl.value].astype(np.int64), hi[:nh.value].astype(np.int64)
