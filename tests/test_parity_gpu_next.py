"""GPU parity of the NEXT rows through the C ABI against the oracle.

NEXT-3: general decoupled kernels (kernel_gamma != d - 2, reading #25): the tables change,
the kernels do not -- Q from fks_collide and F^{n+1} from fks_step within 1e-11 (§8(c.5)).
"""
import numpy as np
import pytest

import workloads
from oracle import collision, step as ostep, tables

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    if not _t.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return _t


@pytest.fixture(scope="module")
def fks():
    from paper_1608_08009_b200 import fks as _f
    return _f


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def rel_err_Q(Qg, f, tab, direct):
    worst = 0.0
    for c in range(f.shape[0]):
        ev = collision.collide_direct if direct else collision.collide_fft
        Q, g, l = ev(f[c], tab, return_parts=True)
        worst = max(worst, np.max(np.abs(Qg[c] - Q)) / np.max(np.abs(g) + np.abs(l)))
    return worst


# ---------------------------------------------------------------- NEXT-3
@pytest.mark.parametrize("gamma", [0.0, 0.5, 2.0, -0.5])
@pytest.mark.parametrize("N,kind", [(8, "random"), (16, "smooth")])
def test_collide_3d_general_gamma(torch, fks, gamma, N, kind):
    """3D VHS with gamma != 1 (3D Maxwell molecules at gamma = 0): decoupled tables, same kernel."""
    L, nc = 7.0, 9
    f = workloads.family(kind, 3, N, L, nc, seed=51)
    ctx = fks.Context(3, 0, [nc], N, L, 24, kernel_gamma=gamma)
    Q = torch.empty(nc, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(3, N, L, gamma=gamma)
    assert rel_err_Q(host(Q), f, tab, direct=(N == 8)) <= TOL


def test_collide_3d_32_maxwell_molecules(torch, fks):
    """N = 32^3 (C2 shape), gamma = 0, more cells than resident groups."""
    N, L, nc = 32, 7.0, 23
    f = workloads.family("random", 3, N, L, nc, seed=52)
    ctx = fks.Context(3, 0, [nc], N, L, 24, kernel_gamma=0.0)
    Q = torch.empty(nc, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(3, N, L, gamma=0.0)
    assert rel_err_Q(host(Q)[:6], f[:6], tab, direct=False) <= TOL


@pytest.mark.parametrize("gamma", [1.0, 2.0, 0.3])
def test_collide_2d_general_gamma(torch, fks, gamma):
    """2D VHS with gamma != 0 against the literal O(n^2) double sum."""
    N, L, nc = 32, 9.0, 7
    f = workloads.family("bkw", 2, N, L, nc, seed=53)
    ctx = fks.Context(2, 0, [nc], N, L, 8, kernel_gamma=gamma)
    Q = torch.empty(nc, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(2, N, L, A=8, gamma=gamma)
    assert rel_err_Q(host(Q), f, tab, direct=True) <= TOL


def test_step_3d_maxwell_molecules_C2_cells(torch, fks):
    """Fused step (a3-a9) of C2 cells with 3D Maxwell molecules (gamma = 0) and the product grid."""
    from oracle import kernels as okern
    c = workloads.config("C2")
    N, L, nc = c["N"], c["L"], 7
    f = workloads.initial_state(c, ncells=nc, start=200)
    ctx = fks.Context(3, 0, [nc], N, L, 64, kernel_gamma=0.0)
    out = torch.empty(nc, N, N, N, dtype=torch.float64, device="cuda")
    ctx.step(dev(torch, f), out, c["dt"])
    ctx.check()
    tab = tables.build_tables(3, N, L, gamma=0.0, directions=okern.directions_3d_product(8, 8))
    ref = ostep.homogeneous_step(f, tab, c["dt"])
    got = host(out)
    for i in range(nc):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))
