"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol the header
declares, its host-built tables and shift tables agree with the independent oracle, and
fks_init refuses to run without an sm_100 device (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import kernels as okern
from oracle import tables as otab
from oracle import transport as otr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fks.h")


@pytest.fixture(scope="module")
def fks():
    from paper_1608_08009_b200 import _lib, fks
    _lib.load()
    return fks


def test_exports_every_header_symbol(fks):
    names = set(re.findall(r"\b(fks_[a-z_]+)\s*\(", open(HEADER).read()))
    assert {"fks_init", "fks_collide", "fks_transport", "fks_step", "fks_moments"} <= names
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1608_08009_b200", "libfks.so"))
    for nm in sorted(names):
        assert hasattr(lib, nm), nm


def test_strerror(fks):
    lib = fks.load()
    for s in range(0, -8, -1):
        assert lib.fks_strerror(s)


@pytest.mark.parametrize("dv,N,L,A,gamma", [(2, 8, 4.0, 8, None), (2, 16, 6.0, 8, None), (2, 32, 9.0, 8, None),
                                            (3, 8, 7.0, 24, None), (3, 16, 7.0, 24, None), (3, 8, 7.0, 64, None),
                                            (3, 16, 7.0, 24, 0.0), (3, 8, 7.0, 24, 0.5), (3, 16, 7.0, 64, 2.0),
                                            (3, 8, 7.0, 24, -0.5), (2, 32, 9.0, 8, 1.0), (2, 16, 6.0, 8, 0.3),
                                            (2, 64, 12.0, 8, None), (3, 64, 7.0, 24, None),
                                            (2, 4, 3.0, 8, None), (3, 4, 4.0, 24, None)])
def test_host_tables_match_oracle(fks, dv, N, L, A, gamma):
    """Two independent table builders (C++ in the library, numpy in the oracle) agree to a few
    ulp: phi/psi (reading #2), directions (reading #17, reading #6),
    symmetrisation (reading #10) and D; for general gamma (NEXT-3, reading #25) the quadrature
    phi_{R,a} (Sturm bisection + Newton in the library, numpy eigvalsh + Newton in the oracle)."""
    al, alp, D, w, e, s = fks.host_tables(dv, N, L, A, kernel_gamma=gamma)
    if dv == 2:
        ref = otab.build_tables(2, N, L, A=A, gamma=gamma)
    elif A == 24:
        ref = otab.build_tables(3, N, L, gamma=gamma)
    else:
        ref = otab.build_tables(3, N, L, directions=okern.directions_3d_product(8, 8), gamma=gamma)
    np.testing.assert_allclose(w, ref.w, rtol=1e-14, atol=0)
    for p in range(A):
        scale = np.abs(ref.alpha[p]).max()
        assert np.max(np.abs(al[p] - ref.alpha[p].reshape(-1))) <= 1e-13 * scale
        scale = np.abs(ref.alphap[p]).max()
        assert np.max(np.abs(alp[p] - ref.alphap[p].reshape(-1))) <= 1e-13 * scale
    assert np.max(np.abs(D - ref.D.reshape(-1))) <= 1e-13 * np.abs(ref.D).max()
    assert abs(s / ref.scale - 1) < 1e-14


def test_design24_directions_match(fks):
    _, _, _, w, e, _ = fks.host_tables(3, 8, 7.0, 24)
    eo, wo = okern.directions_3d_design24()
    # same set of 24 unit vectors (order-independent)
    for v in e:
        assert np.min(np.linalg.norm(eo - v, axis=1)) < 1e-15


def test_host_shift_matches_oracle(fks):
    """a1: delta_k from the same fp64 expression (reading #16), exact equality."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        N = int(rng.choice([8, 16, 32]))
        L = float(rng.uniform(3, 16))
        h = float(rng.uniform(0.003, 0.2))
        dt = h / (L - L / N) * float(rng.uniform(0.2, 1.0))
        n = int(rng.integers(0, 5000))
        got = fks.host_shift(n, N, L, dt, h)
        ref = otr.shift_delta(n, N, L, dt, h)
        np.testing.assert_array_equal(got.astype(np.int64), ref)
        assert set(np.unique(got)) <= {-1, 0, 1}


def test_init_without_gpu_fails_loudly(fks):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(fks.FksError) as ei:
        fks.Context(3, 0, [4], 8, 7.0, 24)
    assert ei.value.status == -4  # FKS_E_CUDA


def test_init_argument_validation(fks):
    """Argument errors are reported before any device work (FKS_E_INVAL / FKS_E_UNSUPPORTED)."""
    with pytest.raises(fks.FksError) as ei:
        fks.Context(3, 0, [4], 12, 7.0, 24)          # N not in {8,16,32,64}
    assert ei.value.status == -1
    with pytest.raises(fks.FksError) as ei:
        fks.Context(3, 0, [4], 8, 7.0, 24, kernel_gamma=2.5)   # outside -1 < gamma <= 2 (reading #25)
    assert ei.value.status == -2
    with pytest.raises(fks.FksError) as ei:
        fks.Context(2, 0, [4], 8, 7.0, 8, kernel_gamma=-1.0)   # phi_{R,a} diverges at gamma = -1
    assert ei.value.status == -2
    with pytest.raises(fks.FksError) as ei:
        fks.Context(3, 0, [4], 8, 7.0, 23)           # no built-in 23-direction set
    assert ei.value.status == -2


@pytest.mark.parametrize("kw,status", [
    (dict(dv=4), -1),                                   # velocity dimension 2 | 3
    (dict(dv=2, dx=3), -1),                             # dx <= dv (axis a shifts with velocity component a)
    (dict(dx=4), -1),
    (dict(dx=-1), -1),
    (dict(Nv=24), -1),                                  # not a power of two in [4, 64]
    (dict(Nv=2), -1),                                   # below the range 4 <= N <= 64
    (dict(Nv=128), -1),                                 # above it
    (dict(L=0.0), -1),
    (dict(L=-3.0), -1),
    (dict(dx=1, M=[0]), -1),                            # empty axis
    (dict(dx=0, M=[0]), -1),
    (dict(dx=1, M=[4], h=0.0), -1),                     # spacing
    (dict(dx=1, M=[4], h=0.1, bc=[5, 0]), -1),          # face kind out of range
    (dict(dx=2, M=[4, 4], h=0.1, bc=[3, 0, 0, 0]), -1),  # HALO on a non-slab axis
    (dict(dx=2, M=[70000, 70000], h=0.1), -1),          # more than 2^31 local cells
    (dict(gamma=-1.0), -2),                             # phi_{R,a} diverges
    (dict(gamma=2.5), -2),
    (dict(A=23), -2),                                   # no built-in 23-direction set in 3D
    (dict(A=0), -2),
])
def test_init_rejects_bad_arguments(fks, kw, status):
    """fks_init validates every argument before touching the device (include/fks.h: argument errors
    return synchronously with nothing created)."""
    a = dict(dv=3, dx=0, M=[4], Nv=8, L=7.0, A=24, gamma=None, h=1.0, bc=None)
    a.update(kw)
    with pytest.raises(fks.FksError) as ei:
        fks.Context(a["dv"], a["dx"], a["M"], a["Nv"], a["L"], a["A"], kernel_gamma=a["gamma"], h=a["h"], bc=a["bc"])
    assert ei.value.status == status


def test_host_entry_points_reject_bad_arguments(fks):
    lib = fks.load()
    import ctypes
    out = (ctypes.c_int8 * 64)()
    n1, n2 = ctypes.c_int(), ctypes.c_int()
    assert lib.fks_host_shift(0, 0, 1.0, 0.1, 0.1, out) == -1          # Nv
    assert lib.fks_host_shift(-1, 8, 1.0, 0.1, 0.1, out) == -1         # n < 0
    assert lib.fks_host_shift(0, 8, 1.0, 0.1, 0.0, out) == -1          # h
    assert lib.fks_host_halo_slices(0, 8, 5.0, 0.5, 0.1, out, ctypes.byref(n1), out, ctypes.byref(n2)) == -2  # |delta| > 1
    assert lib.fks_comm_loopback_create(0, ctypes.byref(ctypes.c_void_p())) == -1
    assert lib.fks_set_scheme(None, 0, 0) == -1
    assert lib.fks_step(None, None, None, 0.1) == -1
    assert lib.fks_finalize(None) == -1
