"""GPU parity of the 3D N = 64 path (kernels3d64.cu: a 64-CTA group per cell, each transform
through L2 twice) and its HBM-bound companions at 64^3, through the C ABI against the oracle.

The velocity grids the paper runs reach 64 points per axis; the 32^3 kernel's
8-CTA group cannot hold a 4 MiB complex 64^3 field, so this size has its own kernel.
"""
import numpy as np
import pytest

import workloads
from oracle import bgk, collision, step as ostep, tables, transport

pytestmark = pytest.mark.gpu
TOL = 1e-11
N, L = 64, 7.0


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


@pytest.fixture(scope="module")
def tab():
    return tables.build_tables(3, N, L)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def test_collide_3d_n64(torch, fks, tab):
    """Q of 6 cells (more than the 4 resident groups: a second, ragged round) against the FFT
    evaluator element by element, and sampled modes of Q^ against the literal O(n) sum per mode
    in Fourier space -- independent of any transform pass order."""
    nc = 6
    f = workloads.family("random", 3, N, L, nc, seed=81)
    ctx = fks.Context(3, 0, [nc], N, L, 24)
    Q = torch.empty(nc, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    Qg = host(Q)
    for c in range(nc):
        ref, g, l = collision.collide_fft(f[c], tab, return_parts=True)
        assert np.max(np.abs(Qg[c] - ref)) <= TOL * np.max(np.abs(g) + np.abs(l)), c
    n = N ** 3
    modes = [0, 1, 3 * N + 5, 63 * N * N + 31 * N + 32, N * N * 32 + N * 32 + 32, n - 1]
    for c in (0, nc - 1):
        Qh, Qgain, Qloss = collision.qhat_direct(f[c], tab, modes)
        got = collision.dft(Qg[c]).reshape(-1)[modes]
        scale = np.max(np.abs(tab.scale * Qgain) + np.abs(tab.scale * Qloss))
        assert np.max(np.abs(got - tab.scale * Qh)) <= 1e-12 * scale


@pytest.mark.parametrize("integ", ["euler", "heun"])
def test_step_3d_n64_homogeneous(torch, fks, tab, integ):
    """Fused step (projection + Euler, or the Heun stages) of 5 cells, two steps; conservation
    of mass, momentum and energy by the projection to round-off."""
    nc, dt, tau = 5, 0.05, 0.7
    f = workloads.family("smooth", 3, N, L, nc, seed=82)
    ctx = fks.Context(3, 0, [nc], N, L, 24)
    ctx.set_params(tau=tau)
    if integ == "heun":
        ctx.set_scheme(fks.SPLIT_LIE, fks.TIME_HEUN)
    a, b = dev(torch, f), torch.empty_like(dev(torch, f))
    ref = f.copy()
    for _ in range(2):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.homogeneous_step(ref, tab, dt, tau=tau, integrator=integ)
    ctx.check()
    got = host(a)
    v = -L + (np.arange(N) + 0.5) * (2 * L / N)
    VZ, VY, VX = np.meshgrid(v, v, v, indexing="ij")
    for i in range(nc):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i
        for w in (np.ones_like(VX), VX, VY, VZ, VX * VX + VY * VY + VZ * VZ):
            m0, m1 = np.sum(f[i] * w), np.sum(got[i] * w)
            assert abs(m1 - m0) <= 1e-12 * np.sum(np.abs(f[i]) * (np.abs(w) + 1)), i


def _spatial(dxd, M, bc, seed):
    rng = np.random.default_rng(400 + seed)
    h = 0.1
    dt = 0.93 * h / (L - L / N)
    shape = tuple(M[::-1]) + (N,) * 3
    base = workloads.family("smooth", 3, N, L, 1, seed=seed)[0]
    F = (base[None] * rng.uniform(0.5, 1.5, int(np.prod(M)))[(...,) + (None,) * 3]).reshape(shape)
    ghosts = {f: workloads.family("smooth", 3, N, L, 1, seed=seed + 10 + f)[0] for f in range(2 * dxd)
              if bc[f] == transport.GHOST}
    return F, h, dt, ghosts


@pytest.mark.parametrize("specular", [False, True])
def test_step_3d_n64_with_transport(torch, fks, tab, specular):
    """1D x 3D at 64^3: ghost / outflow faces, a solid cell (specular walls or not), fused
    transport + collision steps, two steps against the oracle."""
    dxd, M = 1, [5]
    bc = [transport.GHOST, transport.OUTFLOW]
    F, h, dt, ghosts = _spatial(dxd, M, bc, seed=20)
    solid = np.zeros((5,), dtype=bool)
    solid[2] = True
    ctx = fks.Context(3, dxd, M, N, L, 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    if specular:
        ctx.set_specular(True)
    ctx.set_params(tau=0.4)
    cfg = dict(dx_dim=dxd, dv=3, N=N, L=L, dt=dt, dx=h, tau=0.4, bc=bc, ghosts=ghosts, solid=solid,
               specular=specular)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(2):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.step(ref, s, cfg, tab)
    ctx.check()
    got = host(a)
    for i in range(5):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i


def test_n64_3d_transport_moments_bgk(torch, fks):
    """The HBM-bound companions at 64^3: transport bitwise, moments to 1e-13, BGK step to 1e-11."""
    from oracle import moments as omom
    dxd, M = 2, [3, 2]
    bc = [transport.PERIODIC, transport.PERIODIC, transport.GHOST, transport.OUTFLOW]
    F, h, dt, ghosts = _spatial(dxd, M, bc, seed=21)
    ctx = fks.Context(3, dxd, M, N, L, 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ctx.transport(a, b, dt)
    np.testing.assert_array_equal(host(b), transport.gather(F, 0, dxd, 3, N, L, dt, h, bc, ghosts))
    nc = 6
    rho = torch.empty(nc, dtype=torch.float64, device="cuda")
    u = torch.empty(nc, 3, dtype=torch.float64, device="cuda")
    T = torch.empty(nc, dtype=torch.float64, device="cuda")
    ctx.moments(a, rho, u, T)
    ro, uo, To = omom.moments_batch(F.reshape(nc, N, N, N), 3, N, L)
    np.testing.assert_allclose(host(rho), ro, rtol=1e-13)
    np.testing.assert_allclose(host(u), uo, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(host(T), To, rtol=1e-12)
    f0 = workloads.family("random", 3, N, L, 3, seed=22)
    c0 = fks.Context(3, 0, [3], N, L, 24)
    c0.set_params(tau=0.8)
    out = torch.empty_like(dev(torch, f0))
    c0.step_bgk(dev(torch, f0), out, 0.05, bgk.NU_RHO, 0.0)
    ref = bgk.homogeneous_bgk_step(f0, 0.05, 0.8, bgk.NU_RHO, 0.0, 3, N, L)
    got = host(out)
    for i in range(3):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))
