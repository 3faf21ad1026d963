"""GPU parity of the N = 4 path (kernels_small.cu: one thread per velocity point, the transforms as
4-point DFT passes in SMEM) through the C ABI against the oracle -- the low end of the boundary's
range 4 <= N <= 64."""
import numpy as np
import pytest

import workloads
from oracle import bgk, collision, step as ostep, tables, transport

pytestmark = pytest.mark.gpu
TOL = 1e-11
N = 4


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


def _tab(dv, L):
    return tables.build_tables(2, N, L, A=8) if dv == 2 else tables.build_tables(3, N, L)


@pytest.mark.parametrize("dv,L,nc", [(2, 3.0, 37), (3, 4.0, 9)])
def test_collide_n4_vs_literal_sum(torch, fks, dv, L, nc):
    """Q against the literal O(n^2 A) bilinear form on every cell (ragged
    against the 16 / 4 cells per CTA)."""
    f = workloads.family("random", dv, N, L, nc, seed=91)
    ctx = fks.Context(dv, 0, [nc], N, L, 8 if dv == 2 else 24)
    Q = torch.empty((nc,) + (N,) * dv, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = _tab(dv, L)
    Qg = host(Q)
    for c in range(nc):
        ref, g, l = collision.collide_direct(f[c], tab, return_parts=True)
        assert np.max(np.abs(Qg[c] - ref)) <= TOL * np.max(np.abs(g) + np.abs(l)), c


@pytest.mark.parametrize("dv,L", [(2, 3.0), (3, 4.0)])
@pytest.mark.parametrize("integ", ["euler", "heun"])
def test_step_n4_homogeneous(torch, fks, dv, L, integ):
    nc, dt, tau = 21, 0.05, 0.7
    f = workloads.family("smooth", dv, N, L, nc, seed=92)
    ctx = fks.Context(dv, 0, [nc], N, L, 8 if dv == 2 else 24)
    ctx.set_params(tau=tau)
    if integ == "heun":
        ctx.set_scheme(fks.SPLIT_LIE, fks.TIME_HEUN)
    a, b = dev(torch, f), torch.empty_like(dev(torch, f))
    tab = _tab(dv, L)
    ref = f.copy()
    for _ in range(3):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.homogeneous_step(ref, tab, dt, tau=tau, integrator=integ, evaluator="direct")
    ctx.check()
    got = host(a)
    for i in range(nc):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i


@pytest.mark.parametrize("specular,splitting", [(False, "lie"), (True, "lie"), (False, "strang")])
def test_step_n4_with_transport(torch, fks, specular, splitting):
    """2D x 3D at N = 4: ghost / outflow / periodic faces, a solid cell, specular walls, Strang
    splitting; three steps against the oracle."""
    dxd, dv, M, L = 2, 3, [5, 4], 4.0
    bc = [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC]
    rng = np.random.default_rng(93)
    h = 0.1
    dt = 0.9 * h / (L - L / N)
    base = workloads.family("smooth", dv, N, L, 1, seed=93)[0]
    F = (base[None] * rng.uniform(0.5, 1.5, 20)[:, None, None, None]).reshape((4, 5) + (N,) * dv)
    ghosts = {0: workloads.family("smooth", dv, N, L, 1, seed=94)[0]}
    solid = np.zeros((4, 5), dtype=bool)
    solid[2, 2] = True
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    ctx.set_ghost(0, dev(torch, ghosts[0]))
    ctx.set_solid(solid)
    if specular:
        ctx.set_specular(True)
    if splitting == "strang":
        ctx.set_scheme(fks.SPLIT_STRANG, fks.TIME_EULER)
    ctx.set_params(tau=0.5)
    cfg = dict(dx_dim=dxd, dv=dv, N=N, L=L, dt=dt, dx=h, tau=0.5, bc=bc, ghosts=ghosts, solid=solid,
               specular=specular)
    tab = _tab(dv, L)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(3):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.step(ref, s, cfg, tab, splitting=splitting)
    ctx.check()
    got = host(a).reshape(20, -1)
    ref = ref.reshape(20, -1)
    for i in range(20):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i


@pytest.mark.parametrize("dv,L", [(2, 3.0), (3, 4.0)])
def test_n4_transport_moments_bgk(torch, fks, dv, L):
    from oracle import moments as omom
    dxd, M = 1, [7]
    bc = [transport.PERIODIC, transport.OUTFLOW]
    h = 0.1
    dt = 1.7 * h / (L - L / N)  # CFL > 1: the general gather
    F = workloads.family("smooth", dv, N, L, 7, seed=95) * np.linspace(0.5, 1.5, 7)[(slice(None),) + (None,) * dv]
    ctx = fks.Context(dv, dxd, M, N, L, 8 if dv == 2 else 24, h=h, bc=bc)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ctx.transport(a, b, dt)
    np.testing.assert_array_equal(host(b), transport.gather(F, 0, dxd, dv, N, L, dt, h, bc, {}))
    rho = torch.empty(7, dtype=torch.float64, device="cuda")
    u = torch.empty(7, dv, dtype=torch.float64, device="cuda")
    T = torch.empty(7, dtype=torch.float64, device="cuda")
    ctx.moments(a, rho, u, T)
    ro, uo, To = omom.moments_batch(F, dv, N, L)
    np.testing.assert_allclose(host(rho), ro, rtol=1e-13)
    np.testing.assert_allclose(host(T), To, rtol=1e-12)
    c0 = fks.Context(dv, 0, [7], N, L, 8 if dv == 2 else 24)
    c0.set_params(tau=0.8)
    out = torch.empty_like(a)
    c0.step_bgk(a, out, 0.05, bgk.NU_RHO, 0.0)
    ref = bgk.homogeneous_bgk_step(F, 0.05, 0.8, bgk.NU_RHO, 0.0, dv, N, L)
    got = host(out)
    for i in range(7):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))
