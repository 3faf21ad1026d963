"""A/B timing of fks_transport / fks_step on the C4 geometry for two builds of libfks (development aid):
  python tools/ab_transport.py paper_1608_08009_b200/libfks.so paper_1608_08009_b200/libfks_r1.so
Binds only the calls whose signatures are unchanged since round 1 (fks_init, fks_set_ghost,
fks_set_solid, fks_set_stream, fks_transport, fks_step, fks_check), alternating the builds."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1608_08009_b200._lib import FksGrid  # noqa: E402


def open_lib(path):
    lib = ctypes.CDLL(path)
    V = ctypes.c_void_p
    lib.fks_init.argtypes = [ctypes.POINTER(FksGrid), ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                             ctypes.POINTER(V)]
    for nm, args in (("fks_set_ghost", [V, ctypes.c_int, V]), ("fks_set_solid", [V, V]), ("fks_set_stream", [V, V]),
                     ("fks_transport", [V, V, V, ctypes.c_double]), ("fks_step", [V, V, V, ctypes.c_double]),
                     ("fks_check", [V])):
        getattr(lib, nm).argtypes = args
    return lib


def main():
    c = workloads.config("C4")
    N, L, dv, n = c["N"], c["L"], c["dv"], c["N"] ** c["dv"]
    M = list(c["cells"][::-1])
    nc = int(np.prod(M))
    v = torch.from_numpy(workloads.initial_state(c, ncells=1).reshape(-1)[:n].copy()).cuda()
    fa = v.expand(nc, n).contiguous()
    fb = torch.empty_like(fa)
    solid = np.ascontiguousarray(workloads.solid_mask(c).reshape(-1).astype(np.uint8))
    ghost = torch.from_numpy(workloads.ghost_vectors(c)[0]).cuda()
    stream = torch.cuda.current_stream()
    ctxs = []
    for path in sys.argv[1:]:
        lib = open_lib(path)
        g = FksGrid()
        g.dv, g.dx, g.h = dv, 2, c["dx"]
        g.M[0], g.M[1], g.M[2] = M[0], M[1], 1
        for f, b in enumerate(c["bc"] + [0, 0]):
            g.bc[f] = b
        h = ctypes.c_void_p()
        assert lib.fks_init(ctypes.byref(g), N, L, c["A"], 1.0, ctypes.byref(h)) == 0
        assert lib.fks_set_ghost(h, 0, ctypes.c_void_p(ghost.data_ptr())) == 0
        assert lib.fks_set_solid(h, solid.ctypes.data_as(ctypes.c_void_p)) == 0
        lib.fks_set_stream(h, ctypes.c_void_p(stream.cuda_stream))
        ctxs.append((path, lib, h))
    for rnd in range(3):
        for path, lib, h in ctxs:
            for what in ("fks_transport",):
                fn = getattr(lib, what)
                fn(h, ctypes.c_void_p(fa.data_ptr()), ctypes.c_void_p(fb.data_ptr()), c["dt"])
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(10):
                    fn(h, ctypes.c_void_p(fa.data_ptr()), ctypes.c_void_p(fb.data_ptr()), c["dt"])
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                assert lib.fks_check(h) == 0
                print(f"round {rnd} {os.path.basename(path)} {what}: {ms:.3f} ms, {2 * nc * n * 8 / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
