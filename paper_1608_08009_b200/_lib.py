"""ctypes loader for libfks.so (the in-tree sm_100a build).  No fallback: if the library is
missing or cannot be loaded this raises, and every fks_* call fails loudly."""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FKS_LIB_VARIANT=<tag> loads libfks_<tag>.so (an in-tree development build of a kernel variant).
_VARIANT = os.environ.get("FKS_LIB_VARIANT")
LIB_PATH = os.path.join(HERE, f"libfks_{_VARIANT}.so" if _VARIANT else "libfks.so")

c_int, c_int64, c_double, c_void_p = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_DOUBLE = ctypes.POINTER(ctypes.c_double)


class FksGrid(ctypes.Structure):
    """Mirror of fks_grid (include/fks.h)."""
    _fields_ = [("dv", c_int), ("dx", c_int), ("M", c_int64 * 3), ("h", c_double), ("bc", c_int * 6)]


SIGNATURES = {
    "fks_init": (c_int, [ctypes.POINTER(FksGrid), c_int, c_double, c_int, c_double, ctypes.POINTER(c_void_p)]),
    "fks_set_params": (c_int, [c_void_p, c_double, c_double, c_double, c_int]),
    "fks_set_dirs": (c_int, [c_void_p, P_DOUBLE, P_DOUBLE, c_int]),
    "fks_set_ghost": (c_int, [c_void_p, c_int, c_void_p]),
    "fks_set_solid": (c_int, [c_void_p, ctypes.POINTER(ctypes.c_uint8)]),
    "fks_set_halo": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fks_set_stream": (c_int, [c_void_p, c_void_p]),
    "fks_collide": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fks_transport": (c_int, [c_void_p, c_void_p, c_void_p, c_double]),
    "fks_step": (c_int, [c_void_p, c_void_p, c_void_p, c_double]),
    "fks_step_host": (c_int, [c_void_p, c_void_p, c_void_p, c_double]),
    "fks_step_bgk": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_int, c_double]),
    "fks_set_specular": (c_int, [c_void_p, c_int]),
    "fks_set_scheme": (c_int, [c_void_p, c_int, c_int]),
    "fks_comm_unique_id": (c_int, [c_void_p]),
    "fks_ipc_get_handle": (c_int, [c_void_p, c_void_p, ctypes.POINTER(c_int64)]),
    "fks_ipc_open": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "fks_ipc_close": (c_int, [c_void_p]),
    "fks_set_comm": (c_int, [c_void_p, c_void_p, c_int, c_int]),
    "fks_comm_loopback_create": (c_int, [c_int, ctypes.POINTER(c_void_p)]),
    "fks_comm_loopback_destroy": (c_int, [c_void_p]),
    "fks_set_comm_loopback": (c_int, [c_void_p, c_void_p, c_int]),
    "fks_halo_post": (c_int, [c_void_p, c_void_p]),
    "fks_get_comm_stats": (c_int, [c_void_p, ctypes.POINTER(c_int64), ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "fks_moments": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fks_get_state": (c_int, [c_void_p, ctypes.POINTER(c_int64), P_DOUBLE]),
    "fks_set_state": (c_int, [c_void_p, c_int64, c_double]),
    "fks_check": (c_int, [c_void_p]),
    "fks_launch_count": (c_int64, [c_void_p]),
    "fks_finalize": (c_int, [c_void_p]),
    "fks_strerror": (ctypes.c_char_p, [c_int]),
    "fks_host_tables": (c_int, [c_int, c_int, c_double, c_int, c_double, c_double, c_double, P_DOUBLE, P_DOUBLE,
                                P_DOUBLE, P_DOUBLE, P_DOUBLE, P_DOUBLE]),
    "fks_host_shift": (c_int, [c_int64, c_int, c_double, c_double, c_double, ctypes.POINTER(ctypes.c_int8)]),
    "fks_host_halo_slices": (c_int, [c_int64, c_int, c_double, c_double, c_double, ctypes.POINTER(ctypes.c_int8),
                                     ctypes.POINTER(c_int), ctypes.POINTER(ctypes.c_int8), ctypes.POINTER(c_int)]),
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                              "There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


STATUS = {0: "FKS_OK", -1: "FKS_E_INVAL", -2: "FKS_E_UNSUPPORTED", -3: "FKS_E_NOMEM", -4: "FKS_E_CUDA",
          -5: "FKS_E_NCCL", -6: "FKS_E_NONFINITE", -7: "FKS_E_STATE"}


class FksError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = load().fks_strerror(status).decode()
        super().__init__(f"{where}: {STATUS.get(status, status)} ({msg})")


def check(status, where):
    if status != 0:
        raise FksError(status, where)
