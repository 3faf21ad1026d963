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


# ---------------------------------------------------------------- NEXT-4: Heun and Strang
from oracle import bgk, transport  # noqa: E402


def _spatial(dxd, dv, M, N, L, bc, seed):
    rng = np.random.default_rng(300 + seed)
    h = 0.1
    dt = 0.93 * h / (L - L / N)
    shape = tuple(M[::-1]) + (N,) * dv
    base = workloads.family("smooth", dv, N, L, 1, seed=seed)[0]
    F = (base[None] * rng.uniform(0.5, 1.5, int(np.prod(M)))[(...,) + (None,) * dv]).reshape(shape)
    ghosts = {f: workloads.family("smooth", dv, N, L, 1, seed=seed + 10 + f)[0] for f in range(2 * dxd)
              if bc[f] == transport.GHOST}
    return F, h, dt, ghosts


@pytest.mark.parametrize("dv,N,L,A,nc", [(3, 32, 7.0, 24, 5), (2, 32, 9.0, 8, 37), (3, 16, 7.0, 24, 9)])
def test_heun_0d(torch, fks, dv, N, L, A, nc):
    """Heun (RK2) collision integrator on homogeneous cells, three steps, vs the oracle."""
    f = workloads.family("smooth" if dv == 3 else "bkw", dv, N, L, nc, seed=61)
    ctx = fks.Context(dv, 0, [nc], N, L, A)
    ctx.set_params(tau=0.7)
    ctx.set_scheme(fks.SPLIT_LIE, fks.TIME_HEUN)
    a, b = dev(torch, f), torch.empty_like(dev(torch, f))
    tab = tables.build_tables(dv, N, L, A=A) if dv == 2 else tables.build_tables(3, N, L)
    ref = f.copy()
    for _ in range(3):
        ctx.step(a, b, 0.05)
        a, b = b, a
        ref = ostep.homogeneous_step(ref, tab, 0.05, tau=0.7, integrator="heun")
    ctx.check()
    got = host(a)
    for i in range(nc):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


@pytest.mark.parametrize("split,integ", [("lie", "heun"), ("strang", "euler"), ("strang", "heun")])
@pytest.mark.parametrize("dxd,dv,M,N,bc,specular", [
    (1, 3, [9], 8, [transport.GHOST, transport.OUTFLOW], False),
    (2, 2, [6, 5], 16, [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC], False),
    (2, 3, [5, 4], 8, [transport.GHOST, transport.OUTFLOW, transport.OUTFLOW, transport.OUTFLOW], True),
    (3, 3, [3, 3, 3], 8, [transport.PERIODIC] * 2 + [transport.OUTFLOW, transport.GHOST] + [transport.PERIODIC] * 2,
     False),
])
def test_scheme_with_transport(torch, fks, dxd, dv, M, N, bc, specular, split, integ):
    """fks_set_scheme sequences (reading #26) with every face kind, solids and specular walls, three
    steps against the oracle's step(splitting=..., integrator=...)."""
    L = 6.0
    F, h, dt, ghosts = _spatial(dxd, dv, M, N, L, bc, seed=dxd * 3 + dv)
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    solid.reshape(-1)[int(np.prod(M)) // 2] = True
    A = 8 if dv == 2 else 24
    ctx = fks.Context(dv, dxd, M, N, L, A, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    if specular:
        ctx.set_specular(True)
    ctx.set_params(tau=0.4)
    ctx.set_scheme(fks.SPLIT_STRANG if split == "strang" else fks.SPLIT_LIE,
                   fks.TIME_HEUN if integ == "heun" else fks.TIME_EULER)
    tab = tables.build_tables(dv, N, L, A=8) if dv == 2 else tables.build_tables(dv, N, L)
    cfg = dict(dx_dim=dxd, dv=dv, N=N, L=L, dt=dt, dx=h, tau=0.4, bc=bc, ghosts=ghosts, solid=solid,
               specular=specular)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(3):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.step(ref, s, cfg, tab, integrator=integ, splitting=split)
    ctx.check()
    got = host(a).reshape((-1,) + (N,) * dv)
    ref = ref.reshape((-1,) + (N,) * dv)
    for i in range(ref.shape[0]):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i


def test_strang_bgk(torch, fks):
    """Strang splitting of the BGK step (NEXT-2 x NEXT-4): T_half B T_half vs the oracle."""
    dxd, dv, M, N, L = 2, 2, [6, 5], 16, 6.0
    bc = [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC]
    F, h, dt, ghosts = _spatial(dxd, dv, M, N, L, bc, seed=5)
    ctx = fks.Context(dv, dxd, M, N, L, 8, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_params(tau=0.5)
    ctx.set_scheme(fks.SPLIT_STRANG, fks.TIME_EULER)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(2):
        ctx.step_bgk(a, b, dt, bgk.NU_RHO, 0.0)
        a, b = b, a
        d1 = transport.shift_delta_half(2 * s, N, L, dt, h)
        d2 = transport.shift_delta_half(2 * s + 1, N, L, dt, h)
        fs = transport.gather(ref, s, dxd, dv, N, L, dt, h, bc, ghosts, delta=d1)
        mid = np.empty_like(fs)
        for j in range(int(np.prod(M))):
            idx = np.unravel_index(j, tuple(M[::-1]))
            mid[idx] = bgk.bgk_step_cell(fs[idx], dt, 0.5, bgk.NU_RHO, 0.0, dv, N, L)
        ref = transport.gather(mid, s, dxd, dv, N, L, dt, h, bc, ghosts, delta=d2)
    got = host(a).reshape((-1,) + (N,) * dv)
    ref = ref.reshape((-1,) + (N,) * dv)
    for i in range(ref.shape[0]):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


def test_scheme_argument_errors(torch, fks):
    """fks_set_scheme validates its arguments; Strang is refused on a partitioned grid and Heun by
    the BGK step (include/fks.h)."""
    N, L = 8, 7.0
    ctx = fks.Context(3, 0, [2], N, L, 24)
    for sp, it in ((2, 0), (0, 5), (-1, 0)):
        with pytest.raises(fks.FksError) as ei:
            ctx.set_scheme(sp, it)
        assert ei.value.status == -1
    ctx.set_scheme(fks.SPLIT_LIE, fks.TIME_HEUN)
    f = dev(torch, workloads.family("smooth", 3, N, L, 2, seed=6))
    with pytest.raises(fks.FksError) as ei:
        ctx.step_bgk(f, torch.empty_like(f), 0.01, bgk.NU_RHO, 0.0)
    assert ei.value.status == -2
    ctx2 = fks.Context(3, 1, [4], N, L, 24, h=0.1, bc=[fks.BC_HALO, fks.BC_OUTFLOW])
    with pytest.raises(fks.FksError) as ei:
        ctx2.set_scheme(fks.SPLIT_STRANG, fks.TIME_EULER)
    assert ei.value.status == -2
    ctx2.set_scheme(fks.SPLIT_LIE, fks.TIME_HEUN)   # Heun on a partitioned grid is fine


def test_full_size_C3_strang_heun_sampled(torch, fks):
    """BASELINE configs[2] (1Dx3D Sod, 400 cells, Dirichlet ghosts, 32^3) at full size with Strang
    splitting + Heun: one step, sampled cells (both faces, the contact, the interior) against the
    oracle, which computes the collided half-step state only where the second half transport reads."""
    c = workloads.config("C3")
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    M = list(c["cells"][::-1])
    F = workloads.initial_state(c)
    F = F * (1.0 + 0.1 * np.random.default_rng(12).random(F.shape[:1]))[(...,) + (None,) * dv]
    ghosts = workloads.ghost_vectors(c)
    ctx = fks.Context(dv, dxd, M, N, L, A, h=c["dx"], bc=c["bc"])
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_params(tau=c["tau"])
    ctx.set_scheme(fks.SPLIT_STRANG, fks.TIME_HEUN)
    out = torch.empty_like(dev(torch, F))
    ctx.step(dev(torch, F), out, c["dt"])
    ctx.check()
    got = host(out)
    sample = [0, 1, 199, 200, 201, 398, 399]
    need = sorted({j + d for j in sample for d in (-1, 0, 1) if 0 <= j + d < M[0]})
    dt, hx = c["dt"], c["dx"]
    d1 = transport.shift_delta_half(0, N, L, dt, hx)
    d2 = transport.shift_delta_half(1, N, L, dt, hx)
    fs = transport.gather(F, 0, dxd, dv, N, L, dt, hx, c["bc"], ghosts, cells=need, delta=d1)
    tab = tables.build_tables(dv, N, L)
    cfg = dict(dv=dv, N=N, L=L, dt=dt, tau=c["tau"])
    mid = np.full_like(F, np.nan)
    for i, j in enumerate(need):
        mid[j] = ostep._collision_update(fs[i], cfg, tab, collision.collide_fft, "heun")
    ref = transport.gather(mid, 0, dxd, dv, N, L, dt, hx, c["bc"], ghosts, cells=sample, delta=d2)
    for i, j in enumerate(sample):
        assert np.max(np.abs(got[j] - ref[i])) <= TOL * np.max(np.abs(ref[i])), j


# ---------------------------------------------------------------- N = 64 velocity grids (2D)
@pytest.mark.parametrize("kind", ["bkw", "random"])
def test_collide_2d_n64(torch, fks, kind):
    """2D 64^2, pencils split over lane pairs: Q vs the literal double sum (3 cells)
    and vs the FFT evaluator (all 9 cells; ragged against the 2 cells per CTA)."""
    N, L, nc = 64, 12.0, 9
    f = workloads.family(kind, 2, N, L, nc, seed=71)
    ctx = fks.Context(2, 0, [nc], N, L, 8)
    Q = torch.empty(nc, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(2, N, L, A=8)
    Qg = host(Q)
    assert rel_err_Q(Qg[:2], f[:2], tab, direct=True) <= TOL
    assert rel_err_Q(Qg, f, tab, direct=False) <= TOL


@pytest.mark.parametrize("integ", ["euler", "heun"])
def test_step_2d_n64_with_transport(torch, fks, integ):
    """Fused steps on a 1D x 2D grid at N = 64 (ghost / outflow faces, a solid cell), both
    integrators, three steps against the oracle."""
    dxd, dv, M, N, L = 1, 2, [7], 64, 12.0
    bc = [transport.GHOST, transport.OUTFLOW]
    F, h, dt, ghosts = _spatial(dxd, dv, M, N, L, bc, seed=8)
    solid = np.zeros((7,), dtype=bool)
    solid[3] = True
    ctx = fks.Context(dv, dxd, M, N, L, 8, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    ctx.set_params(tau=0.4)
    if integ == "heun":
        ctx.set_scheme(fks.SPLIT_LIE, fks.TIME_HEUN)
    tab = tables.build_tables(2, N, L, A=8)
    cfg = dict(dx_dim=dxd, dv=dv, N=N, L=L, dt=dt, dx=h, tau=0.4, bc=bc, ghosts=ghosts, solid=solid)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(3):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.step(ref, s, cfg, tab, integrator=integ)
    ctx.check()
    got = host(a)
    for i in range(7):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i


def test_n64_transport_moments_bgk(torch, fks):
    """The HBM-bound companions at N = 64: transport bitwise, moments to 1e-13, BGK step to 1e-11."""
    from oracle import moments as omom
    dxd, dv, M, N, L = 2, 2, [4, 3], 64, 12.0
    bc = [transport.PERIODIC, transport.PERIODIC, transport.GHOST, transport.OUTFLOW]
    F, h, dt, ghosts = _spatial(dxd, dv, M, N, L, bc, seed=9)
    ctx = fks.Context(dv, dxd, M, N, L, 8, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ctx.transport(a, b, dt)
    np.testing.assert_array_equal(host(b), transport.gather(F, 0, dxd, dv, N, L, dt, h, bc, ghosts))
    nc = 12
    rho = torch.empty(nc, dtype=torch.float64, device="cuda")
    u = torch.empty(nc, 2, dtype=torch.float64, device="cuda")
    T = torch.empty(nc, dtype=torch.float64, device="cuda")
    ctx.moments(a, rho, u, T)
    ro, uo, To = omom.moments_batch(F.reshape(nc, N, N), dv, N, L)
    np.testing.assert_allclose(host(rho), ro, rtol=1e-13)
    np.testing.assert_allclose(host(T), To, rtol=1e-12)
    f0 = workloads.family("random", 2, N, L, 5, seed=3)
    c0 = fks.Context(2, 0, [5], N, L, 8)
    c0.set_params(tau=0.8)
    out = torch.empty_like(dev(torch, f0))
    c0.step_bgk(dev(torch, f0), out, 0.05, bgk.NU_RHO, 0.0)
    ref = bgk.homogeneous_bgk_step(f0, 0.05, 0.8, bgk.NU_RHO, 0.0, 2, N, L)
    got = host(out)
    for i in range(5):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


@pytest.mark.parametrize("specular,cfl", [(False, 0.93), (True, 0.93), (False, 1.6)])
def test_bgk_3d_n32_with_transport(torch, fks, specular, cfl):
    """NEXT-2 at 32^3 with transport (the TMEM-resident k_bgk_tmem32: f* parked in tensor memory
    between the moment pass and the update pass): ghost / outflow faces, a solid cell, specular
    walls, CFL > 1 (general gather), two steps against the oracle."""
    dxd, dv, M, N, L = 2, 3, [3, 3], 32, 8.0
    bc = [transport.GHOST, transport.OUTFLOW, transport.OUTFLOW, transport.PERIODIC]
    F, h, _, ghosts = _spatial(dxd, dv, M, N, L, bc, seed=12)
    dt = cfl * h / (L - L / N)
    solid = np.zeros((3, 3), dtype=bool)
    solid[1, 1] = True
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    if specular:
        ctx.set_specular(True)
    ctx.set_params(tau=0.5)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(2):
        ctx.step_bgk(a, b, dt, bgk.NU_RHO, 0.0)
        a, b = b, a
        if specular:
            fs = transport.gather_specular(ref, s, dxd, dv, N, L, dt, h, bc, ghosts, solid)
        else:
            fs = transport.gather(ref, s, dxd, dv, N, L, dt, h, bc, ghosts)
        nxt = np.empty_like(ref)
        for j in range(9):
            idx = np.unravel_index(j, (3, 3))
            nxt[idx] = ref[idx] if solid[idx] else bgk.bgk_step_cell(fs[idx], dt, 0.5, bgk.NU_RHO, 0.0, dv, N, L)
        ref = nxt
    ctx.check()
    got = host(a).reshape((-1,) + (N,) * dv)
    ref = ref.reshape((-1,) + (N,) * dv)
    for i in range(9):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), i
