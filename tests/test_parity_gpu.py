"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Criteria:
  Q from fks_collide:   per cell max_k |Q_gpu - Q_orc| / max_k (|Q+_orc| + |Q-_orc|) <= 1e-11
  F^{n+1} from fks_step: per cell max_k |f_gpu - f_orc| / max_k |f_orc|             <= 1e-11
  transport:            bitwise; moments: 1e-13 relative.
The oracle evaluator is `collide_direct` (the literal O(n^2) bilinear form) wherever it finishes
in seconds and `collide_fft` (pinned to it, tests/test_oracle_pins.py P4) elsewhere.
"""
import numpy as np
import pytest

import workloads
from oracle import bgk, collision, grid, moments, projection, step as ostep, tables, transport

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
    """Per-cell parity norm of §8(c.5)."""
    worst = 0.0
    for c in range(f.shape[0]):
        ev = collision.collide_direct if direct else collision.collide_fft
        Q, g, l = ev(f[c], tab, return_parts=True)
        worst = max(worst, np.max(np.abs(Qg[c] - Q)) / np.max(np.abs(g) + np.abs(l)))
    return worst


# ---------------------------------------------------------------- a4-a7: collide
@pytest.mark.parametrize("N,L", [(8, 4.0), (16, 6.0), (32, 9.0)])
@pytest.mark.parametrize("kind", ["smooth", "neareq", "random", "bkw"])
def test_collide_2d(torch, fks, N, L, kind):
    ncells = 13 if N < 32 else 7          # ragged against the cells-per-CTA grouping
    f = workloads.family(kind, 2, N, L, ncells, seed=1)
    ctx = fks.Context(2, 0, [ncells], N, L, 8)
    Q = torch.empty(ncells, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(2, N, L, A=8)
    assert rel_err_Q(host(Q), f, tab, direct=True) <= TOL


@pytest.mark.parametrize("N,L", [(8, 7.0), (16, 7.0)])
@pytest.mark.parametrize("kind", ["smooth", "neareq", "random"])
def test_collide_3d_small(torch, fks, N, L, kind):
    ncells = 11
    f = workloads.family(kind, 3, N, L, ncells, seed=2)
    ctx = fks.Context(3, 0, [ncells], N, L, 24)
    Q = torch.empty(ncells, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(3, N, L)
    assert rel_err_Q(host(Q), f, tab, direct=(N == 8)) <= TOL


def test_collide_3d_product_directions(torch, fks):
    """The (theta, phi) product grid of P:527-540 (A1 = A2 = 8, reading #6)."""
    from oracle import kernels as okern
    N, L, ncells = 8, 7.0, 5
    f = workloads.family("random", 3, N, L, ncells, seed=3)
    ctx = fks.Context(3, 0, [ncells], N, L, 64)
    Q = torch.empty(ncells, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    tab = tables.build_tables(3, N, L, directions=okern.directions_3d_product(8, 8))
    assert rel_err_Q(host(Q), f, tab, direct=True) <= TOL


@pytest.mark.parametrize("kind", ["smooth", "random", "neareq"])
def test_collide_3d_32(torch, fks, kind):
    """N = 32^3, 24-design (C2 shape), more cells than resident clusters (ragged tail)."""
    N, L = 32, 7.0
    ncells = 37
    f = workloads.family(kind, 3, N, L, ncells, seed=4)
    ctx = fks.Context(3, 0, [ncells], N, L, 24)
    Q = torch.empty(ncells, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    ctx.check()
    tab = tables.build_tables(3, N, L)
    Qg = host(Q)
    assert rel_err_Q(Qg[:12], f[:12], tab, direct=False) <= TOL
    # one cell against modes of the literal double sum, computed one by one
    modes = np.random.default_rng(0).choice(N ** 3, size=4, replace=False)
    qh, _, ql = collision.qhat_direct(f[0], tab, modes=modes)
    _, _, lf = collision.collide_fft(f[0], tab, return_parts=True)
    got = (collision.dft(Qg[0]) / tab.scale).reshape(-1)[modes]
    assert np.max(np.abs(got - qh)) <= TOL * np.max(np.abs(collision.dft(lf) / tab.scale))


# ---------------------------------------------------------------- a3-a9: step
def test_step_0d_3d_C2_cells(torch, fks):
    c = workloads.config("C2")
    N, L = c["N"], c["L"]
    f = workloads.initial_state(c, ncells=19)
    ctx = fks.Context(3, 0, [19], N, L, 24)
    fin, fout = dev(torch, f), torch.empty(19, N, N, N, dtype=torch.float64, device="cuda")
    ctx.step(fin, fout, c["dt"])
    ctx.check()
    tab = tables.build_tables(3, N, L)
    ref = ostep.homogeneous_step(f, tab, c["dt"])
    got = host(fout)
    for i in range(19):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))
    assert ctx.get_state()[0] == 1


def test_step_0d_2d_C1_ten_steps(torch, fks):
    """C1 literal run shape: BKW cells, 10 steps, growth of the difference reported (<= 1e-11)."""
    c = workloads.config("C1")
    N, L = c["N"], c["L"]
    f = workloads.initial_state(c, ncells=7)
    ctx = fks.Context(2, 0, [7], N, L, 8)
    a, b = dev(torch, f), torch.empty(7, N, N, dtype=torch.float64, device="cuda")
    tab = tables.build_tables(2, N, L, A=8)
    ref = f.copy()
    for s in range(10):
        ctx.step(a, b, c["dt"])
        a, b = b, a
        ref = ostep.homogeneous_step(ref, tab, c["dt"])
    got = host(a)
    for i in range(7):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


def _spatial_case(dxd, dv, M, N, L, bc, solid=None, seed=0):
    rng = np.random.default_rng(100 + seed)
    vmax = L - L / N
    h = 0.1
    dt = 0.93 * h / vmax
    shape = tuple(M[::-1]) + (N,) * dv
    base = workloads.family("smooth", dv, N, L, 1, seed=seed)[0]
    F = base[None] * rng.uniform(0.5, 1.5, int(np.prod(M)))[(...,) + (None,) * dv]
    F = F.reshape(shape)
    ghosts = {f: workloads.family("smooth", dv, N, L, 1, seed=seed + 10 + f)[0] for f in range(2 * dxd)
              if bc[f] == transport.GHOST}
    return F, h, dt, ghosts


@pytest.mark.parametrize("dxd,dv,M,N,bc", [
    (1, 3, [12], 8, [transport.GHOST, transport.GHOST]),
    (1, 2, [9], 16, [transport.PERIODIC, transport.PERIODIC]),
    (2, 2, [5, 4], 8, [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC]),
    (2, 3, [4, 3], 8, [transport.GHOST, transport.OUTFLOW, transport.OUTFLOW, transport.OUTFLOW]),
    (3, 3, [3, 3, 3], 8, [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC,
                          transport.OUTFLOW, transport.OUTFLOW]),
])
def test_step_with_transport(torch, fks, dxd, dv, M, N, bc):
    """Three fused steps (a1..a9) with every face kind, against the oracle's split step."""
    L = 6.0
    F, h, dt, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=dxd + dv)
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    if int(np.prod(M)) > 8:
        solid.reshape(-1)[int(np.prod(M)) // 2] = True
    ctx = fks.Context(dv, dxd, M, N, L, 8 if dv == 2 else 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    tab = tables.build_tables(dv, N, L, A=8) if dv == 2 else tables.build_tables(dv, N, L)
    cfg = dict(dx_dim=dxd, dv=dv, N=N, L=L, dt=dt, dx=h, tau=1.0, bc=bc, ghosts=ghosts, solid=solid)
    ref = F.copy()
    for s in range(3):
        ctx.step(a, b, dt)
        a, b = b, a
        ref = ostep.step(ref, s, cfg, tab)
    got = host(a)
    flat_g = got.reshape((-1,) + (N,) * dv)
    flat_r = ref.reshape((-1,) + (N,) * dv)
    for i in range(flat_r.shape[0]):
        assert np.max(np.abs(flat_g[i] - flat_r[i])) <= TOL * np.max(np.abs(flat_r[i]))


@pytest.mark.parametrize("dxd,dv,M,N,bc", [
    (1, 3, [7], 8, [transport.GHOST, transport.OUTFLOW]),
    (2, 2, [6, 5], 16, [transport.PERIODIC, transport.PERIODIC, transport.GHOST, transport.OUTFLOW]),
    (3, 3, [4, 3, 2], 8, [transport.PERIODIC] * 2 + [transport.OUTFLOW, transport.GHOST] + [transport.PERIODIC] * 2),
])
def test_transport_bitwise(torch, fks, dxd, dv, M, N, bc):
    """a1 + a3 alone: a permutation with boundary values, bitwise equal to the oracle over 7 steps."""
    L = 5.0
    F, h, dt, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=7)
    ctx = fks.Context(dv, dxd, M, N, L, 8 if dv == 2 else 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(7):
        ctx.transport(a, b, dt)
        a, b = b, a
        ref = transport.gather(ref, s, dxd, dv, N, L, dt, h, bc, ghosts)
    np.testing.assert_array_equal(host(a), ref)


@pytest.mark.parametrize("cfl", [1.7, 2.6])
def test_transport_bitwise_cfl_above_one(torch, fks, cfl):
    """Shifts of 2-3 cells per step (CFL > 1) take the general gather kernel: still bitwise."""
    dxd, dv, M, N, L = 2, 3, [6, 5], 8, 5.0
    bc = [transport.PERIODIC, transport.PERIODIC, transport.GHOST, transport.OUTFLOW]
    F, h, _, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=11)
    dt = cfl * h / (L - L / N)
    assert np.max(np.abs(transport.shift_delta(0, N, L, dt, h))) >= 2
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(4):
        ctx.transport(a, b, dt)
        a, b = b, a
        ref = transport.gather(ref, s, dxd, dv, N, L, dt, h, bc, ghosts)
    np.testing.assert_array_equal(host(a), ref)


@pytest.mark.parametrize("N,L,ncells", [(16, 6.0, 23), (32, 9.0, 9)])
def test_collide_3d_one_group_many_cells(torch, fks, N, L, ncells, monkeypatch):
    """One CTA group walks every cell: the exchange ring wraps many times, the f* cache parity and
    the next-cell forward overlap are exercised on every cell boundary."""
    monkeypatch.setenv("FKS_MAX_CLUSTERS", "1")
    f = workloads.family("random", 3, N, L, ncells, seed=21)
    ctx = fks.Context(3, 0, [ncells], N, L, 24)
    Q = torch.empty(ncells, N, N, N, dtype=torch.float64, device="cuda")
    ctx.collide(dev(torch, f), Q)
    tab = tables.build_tables(3, N, L)
    assert rel_err_Q(host(Q), f, tab, direct=False) <= TOL
    # and the fused step on the same single group (projection reduction, Euler, TMEM f* cache)
    c = workloads.config("C2")
    g = torch.empty_like(Q)
    ctx.step(dev(torch, f), g, c["dt"])
    ref = ostep.homogeneous_step(f, tab, c["dt"])
    got = host(g)
    for i in range(ncells):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


# ---------------------------------------------------------------- NEXT-1: specular reflection
def _solid_block(M, cells):
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    for c in cells:
        solid[tuple(reversed(c))] = True
    return solid


@pytest.mark.parametrize("dxd,dv,M,N,bc,cells,cfl", [
    (1, 3, [9], 8, [transport.PERIODIC] * 2, [(4,)], 0.93),
    (2, 2, [6, 6], 16, [transport.PERIODIC] * 4, [(2, 2), (3, 2), (2, 3)], 0.93),
    (2, 3, [6, 5], 8, [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC],
     [(2, 1), (2, 2)], 0.93),
    (3, 3, [4, 4, 3], 8, [transport.PERIODIC] * 6, [(1, 1, 1), (2, 1, 1), (1, 2, 1)], 0.93),
    (2, 2, [7, 6], 8, [transport.PERIODIC] * 4, [(3, 3)], 1.8),    # CFL > 1: general gather
])
def test_transport_specular_bitwise(torch, fks, dxd, dv, M, N, bc, cells, cfl):
    """fks_transport with specular reflection = the oracle's gather_specular, bitwise, 5 steps."""
    L = 5.0
    F, h, _, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=13)
    dt = cfl * h / (L - L / N)
    solid = _solid_block(M, cells)
    ctx = fks.Context(dv, dxd, M, N, L, 8 if dv == 2 else 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    ctx.set_specular(True)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(5):
        ctx.transport(a, b, dt)
        a, b = b, a
        ref = transport.gather_specular(ref, s, dxd, dv, N, L, dt, h, bc, ghosts, solid)
    np.testing.assert_array_equal(host(a), ref)


@pytest.mark.parametrize("model", ["boltzmann", "bgk"])
def test_step_specular(torch, fks, model):
    """Fused steps with specular reflection (3D kernel's per-cell source table with mirrored
    components; BGK kernel) against the oracle's gather_specular followed by its collision."""
    dxd, dv, M, N, L = 2, 3, [5, 4], 8, 6.0
    bc = [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC]
    F, h, dt, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=17)
    solid = _solid_block(M, [(2, 1), (2, 2)])
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    ctx.set_specular(True)
    ctx.set_params(tau=0.5)
    tab = tables.build_tables(dv, N, L)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(2):
        if model == "bgk":
            ctx.step_bgk(a, b, dt, bgk.NU_RHO, 0.0)
        else:
            ctx.step(a, b, dt)
        a, b = b, a
        fstar = transport.gather_specular(ref, s, dxd, dv, N, L, dt, h, bc, ghosts, solid)
        nxt = np.empty_like(ref)
        for j in range(int(np.prod(M))):
            idx = np.unravel_index(j, tuple(M[::-1]))
            if solid[idx]:
                nxt[idx] = ref[idx]
            elif model == "bgk":
                nxt[idx] = bgk.bgk_step_cell(fstar[idx], dt, 0.5, bgk.NU_RHO, 0.0, dv, N, L)
            else:
                Q = projection.project_zero_moments(collision.collide_fft(fstar[idx], tab), dv, N, L)
                nxt[idx] = fstar[idx] + (dt / 0.5) * Q
        ref = nxt
    got = host(a).reshape((-1,) + (N,) * dv)
    ref = ref.reshape((-1,) + (N,) * dv)
    for i in range(ref.shape[0]):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


def test_reentry_inflow_schedule_with_specular_solids(torch, fks):
    """NEXT-1 together: the time-dependent inflow of eq. BCs through fks_set_ghost every step and
    specular reflection at a solid box, fused steps vs the oracle with the same ghosts per step."""
    dxd, dv, M, N, L = 2, 3, [6, 5], 8, 6.0
    bc = [transport.GHOST, transport.OUTFLOW, transport.OUTFLOW, transport.OUTFLOW]
    F, h, dt, _ = _spatial_case(dxd, dv, M, N, L, bc, seed=23)
    c = dict(dv=dv, N=N, L=L)
    solid = _solid_block(M, [(3, 2)])
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    ctx.set_solid(solid)
    ctx.set_specular(True)
    ctx.set_params(tau=0.5)
    tab = tables.build_tables(dv, N, L)
    t0 = 1.5 - dt                                   # the inflow starts turning during the run
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(3):
        g = workloads.reentry_inflow_ghost(c, t0 + s * dt)
        ctx.set_ghost(0, dev(torch, g))
        ctx.step(a, b, dt)
        a, b = b, a
        fstar = transport.gather_specular(ref, s, dxd, dv, N, L, dt, h, bc, {0: g}, solid)
        nxt = np.empty_like(ref)
        for j in range(int(np.prod(M))):
            idx = np.unravel_index(j, tuple(M[::-1]))
            if solid[idx]:
                nxt[idx] = ref[idx]
            else:
                Q = projection.project_zero_moments(collision.collide_fft(fstar[idx], tab), dv, N, L)
                nxt[idx] = fstar[idx] + (dt / 0.5) * Q
        ref = nxt
    got = host(a).reshape((-1,) + (N,) * dv)
    ref = ref.reshape((-1,) + (N,) * dv)
    for i in range(ref.shape[0]):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


# ---------------------------------------------------------------- NEXT-2: BGK step
@pytest.mark.parametrize("dv,N,L,kind", [(2, 32, 9.0, "bkw"), (2, 16, 6.0, "random"), (3, 16, 7.0, "smooth"),
                                         (3, 32, 7.0, "random")])
@pytest.mark.parametrize("nu_rule,mu", [(bgk.NU_RHO, 0.0), (bgk.NU_CONST, 1.7), (bgk.NU_EULER, 0.0)])
def test_bgk_step_0d(torch, fks, dv, N, L, kind, nu_rule, mu):
    ncells = 9 if dv == 3 else 37
    f = workloads.family(kind, dv, N, L, ncells, seed=41)
    ctx = fks.Context(dv, 0, [ncells], N, L, 8 if dv == 2 else 24)
    ctx.set_params(tau=0.8)
    out = torch.empty_like(dev(torch, f))
    dt = 0.05
    ctx.step_bgk(dev(torch, f), out, dt, nu_rule, mu)
    ctx.check()
    ref = bgk.homogeneous_bgk_step(f, dt, 0.8, nu_rule, mu, dv, N, L)
    got = host(out)
    for i in range(ncells):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


@pytest.mark.parametrize("dxd,dv,M,N,bc", [
    (1, 3, [9], 8, [transport.GHOST, transport.OUTFLOW]),
    (2, 2, [5, 4], 16, [transport.GHOST, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC]),
])
def test_bgk_step_with_transport(torch, fks, dxd, dv, M, N, bc):
    """Two fused BGK steps (gather + conservative Maxwellian + Euler) with ghosts and a solid cell,
    against the oracle's transport followed by its per-cell BGK step."""
    L = 6.0
    F, h, dt, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=3)
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    solid.reshape(-1)[int(np.prod(M)) // 2] = True
    ctx = fks.Context(dv, dxd, M, N, L, 8 if dv == 2 else 24, h=h, bc=bc)
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    ctx.set_params(tau=0.5)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    vshape = (N,) * dv
    for s in range(2):
        ctx.step_bgk(a, b, dt, bgk.NU_RHO, 0.0)
        a, b = b, a
        fstar = transport.gather(ref, s, dxd, dv, N, L, dt, h, bc, ghosts)
        nxt = np.empty_like(ref)
        for j in range(int(np.prod(M))):
            idx = np.unravel_index(j, tuple(M[::-1]))
            nxt[idx] = ref[idx] if solid[idx] else bgk.bgk_step_cell(fstar[idx], dt, 0.5, bgk.NU_RHO, 0.0, dv, N, L)
        ref = nxt
    got = host(a).reshape((-1,) + vshape)
    ref = ref.reshape((-1,) + vshape)
    for i in range(ref.shape[0]):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i]))


# ---------------------------------------------------------------- a10, flags, determinism, e2e
def test_moments(torch, fks):
    for dv, N, L in [(2, 32, 9.0), (3, 16, 7.0)]:
        f = workloads.family("smooth", dv, N, L, 6, seed=5)
        ctx = fks.Context(dv, 0, [6], N, L, 8 if dv == 2 else 24)
        rho = torch.empty(6, dtype=torch.float64, device="cuda")
        u = torch.empty(6, dv, dtype=torch.float64, device="cuda")
        T = torch.empty(6, dtype=torch.float64, device="cuda")
        ctx.moments(dev(torch, f), rho, u, T)
        ro, uo, To = moments.moments_batch(f, dv, N, L)
        np.testing.assert_allclose(host(rho), ro, rtol=1e-13)
        np.testing.assert_allclose(host(u), uo, rtol=1e-12, atol=1e-13 * np.abs(uo).max())
        np.testing.assert_allclose(host(T), To, rtol=1e-12)


def test_nonfinite_flag(torch, fks):
    N, L = 8, 7.0
    f = workloads.family("smooth", 3, N, L, 3, seed=6)
    f[1, 2, 3, 4] = np.nan
    ctx = fks.Context(3, 0, [3], N, L, 24)
    out = torch.empty(3, N, N, N, dtype=torch.float64, device="cuda")
    ctx.step(dev(torch, f), out, 0.01)
    with pytest.raises(fks.FksError) as ei:
        ctx.check()
    assert ei.value.status == -6
    ctx.check()  # flag cleared


def test_next_entry_points_argument_errors(torch, fks):
    """fks_step_bgk / fks_set_specular reject bad arguments synchronously (include/fks.h)."""
    N, L = 8, 7.0
    f = workloads.family("smooth", 3, N, L, 2, seed=6)
    ctx = fks.Context(3, 0, [2], N, L, 24)
    out = torch.empty(2, N, N, N, dtype=torch.float64, device="cuda")
    for rule, mu in ((7, 0.0), (bgk.NU_CONST, 0.0), (bgk.NU_CONST, -1.0)):
        with pytest.raises(fks.FksError) as ei:
            ctx.step_bgk(dev(torch, f), out, 0.01, rule, mu)
        assert ei.value.status == -1  # FKS_E_INVAL
    # specular reflection on a partitioned grid needs the library exchange (the neighbours' solid
    # flags): with caller-owned halo planes the step is refused
    ctx2 = fks.Context(3, 1, [4], N, L, 24, h=0.1, bc=[fks.BC_HALO, fks.BC_OUTFLOW])
    ctx2.set_solid(np.array([0, 1, 0, 0], dtype=bool))
    ctx2.set_specular(True)
    f4 = dev(torch, workloads.family("smooth", 3, N, L, 4, seed=6))
    ctx2.set_halo(f4[:1].contiguous(), None)
    with pytest.raises(fks.FksError) as ei:
        ctx2.step(f4, torch.empty_like(f4), 0.01)
    assert ei.value.status == -2  # FKS_E_UNSUPPORTED
    ctx2.set_specular(False)
    ctx2.step(f4, torch.empty_like(f4), 0.01)


def test_deterministic_and_host_path(torch, fks):
    """Two runs are bitwise identical; fks_step_host (host buffers) equals the device path."""
    c = workloads.config("C2")
    N, L = c["N"], c["L"]
    f = workloads.initial_state(c, ncells=21)
    outs = []
    for _ in range(2):
        ctx = fks.Context(3, 0, [21], N, L, 24)
        o = torch.empty(21, N, N, N, dtype=torch.float64, device="cuda")
        ctx.step(dev(torch, f), o, c["dt"])
        outs.append(host(o))
    np.testing.assert_array_equal(outs[0], outs[1])
    ctx = fks.Context(3, 0, [21], N, L, 24)
    hin = torch.from_numpy(f.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ctx.step_host(hin, hout, c["dt"])
    np.testing.assert_array_equal(hout.numpy(), outs[0])


@pytest.mark.parametrize("dv,N,ncells", [(3, 8, 311), (2, 16, 5003)])
def test_host_path_pipelined_chunks(torch, fks, dv, N, ncells):
    """fks_step_host on a batch that spans several copy/compute chunks (ragged last chunk) is
    bitwise the device fks_step."""
    L = 6.0
    f = workloads.family("smooth", dv, N, L, ncells, seed=31)
    A = 24 if dv == 3 else 8
    ctx = fks.Context(dv, 0, [ncells], N, L, A)
    o = torch.empty((ncells,) + (N,) * dv, dtype=torch.float64, device="cuda")
    ctx.step(dev(torch, f), o, 0.05)
    ctx_h = fks.Context(dv, 0, [ncells], N, L, A)
    hin = torch.from_numpy(f.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ctx_h.step_host(hin, hout, 0.05)
    np.testing.assert_array_equal(hout.numpy(), host(o))


def test_full_size_C2_launch_sampled(torch, fks):
    """BASELINE configs[1] at full size (4096 cells) in bench.py's launch configuration; sampled
    cells against the oracle one by one, plus exact mass conservation on every cell."""
    c = workloads.config("C2")
    N, L, nc = c["N"], c["L"], c["cells"][0]
    f = workloads.initial_state(c)
    ctx = fks.Context(3, 0, [nc], N, L, 24)
    fin = dev(torch, f)
    out = torch.empty_like(fin)
    ctx.step(fin, out, c["dt"])
    ctx.check()
    tab = tables.build_tables(3, N, L)
    got = host(out)
    for i in [0, 1, 1777, nc - 1]:
        ref = ostep.homogeneous_step(f[i:i + 1], tab, c["dt"])[0]
        assert np.max(np.abs(got[i] - ref)) <= TOL * np.max(np.abs(ref))
    mass_in = f.reshape(nc, -1).sum(axis=1)
    mass_out = got.reshape(nc, -1).sum(axis=1)
    assert np.max(np.abs(mass_out - mass_in) / mass_in) < 1e-12


@pytest.mark.parametrize("dxd,dv,M,N,bc,world", [
    (1, 3, [11], 8, [transport.GHOST, transport.GHOST], 3),
    (2, 3, [4, 7], 8, [transport.GHOST, transport.OUTFLOW, transport.OUTFLOW, transport.OUTFLOW], 2),
    (2, 2, [5, 6], 16, [transport.PERIODIC, transport.PERIODIC, transport.PERIODIC, transport.PERIODIC], 3),
    (3, 3, [3, 2, 5], 8, [transport.OUTFLOW, transport.OUTFLOW, transport.PERIODIC, transport.PERIODIC,
                          transport.GHOST, transport.OUTFLOW], 2),
])
def test_slab_partition_bitwise(torch, fks, dxd, dv, M, N, bc, world):
    """a2: the slab-decomposed step (HALO faces fed with the neighbours' boundary planes) equals
    the single-domain step bitwise, every step (ranks emulated one after another on one GPU;
    the exchange itself is covered by tests/test_parallel_cpu.py)."""
    from paper_1608_08009_b200 import parallel
    L = 6.0
    F, h, dt, ghosts = _spatial_case(dxd, dv, M, N, L, bc, seed=21)
    n = N ** dv
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    solid.reshape(-1)[len(solid.reshape(-1)) // 3] = True
    A = 8 if dv == 2 else 24
    ref_ctx = fks.Context(dv, dxd, M, N, L, A, h=h, bc=bc)
    for face, g in ghosts.items():
        ref_ctx.set_ghost(face, dev(torch, g))
    ref_ctx.set_solid(solid)
    slabs = [parallel.decompose(dxd, M, bc, world, r) for r in range(world)]
    ctxs = []
    for s in slabs:
        c = fks.Context(dv, dxd, list(s.M_local), N, L, A, h=h, bc=s.local_bc(bc))
        for face, g in ghosts.items():
            c.set_ghost(face, dev(torch, g))
        c.set_solid(parallel.local_slice(s, solid.reshape(-1)))
        ctxs.append(c)
    G = dev(torch, F).reshape(-1, n)
    for step in range(3):
        out = torch.empty_like(G)
        ref_ctx.step(G, out, dt)
        for s, c in zip(slabs, ctxs):
            lo, hi = parallel.halos_from_global(s, G)
            c.set_halo(lo.contiguous() if lo is not None else None, hi.contiguous() if hi is not None else None)
            loc = parallel.local_slice(s, G).contiguous()
            o = torch.empty_like(loc)
            c.step(loc, o, dt)
            assert torch.equal(o, parallel.local_slice(s, out)), (step, s.rank)
        G = out


@pytest.mark.parametrize("name,sample", [("C3", [0, 1, 199, 200, 398, 399]),
                                         ("C4", [0, 99, 4236, 4237, 5050, 9999])])
def test_full_size_spatial_sampled(torch, fks, name, sample):
    """BASELINE configs C3 (1Dx3D Sod, 400 cells, Dirichlet ghosts) and C4 (2Dx3D, 100^2 cells,
    inflow/outflow, solid boxes) at full size in bench.py's launch configuration: one fused step,
    sampled cells (faces, interior, next to the solids) against the oracle cell by cell."""
    from oracle import projection as oproj
    c = workloads.config(name)
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    M = list(c["cells"][::-1])
    F = workloads.initial_state(c)
    if name == "C4":  # break the uniformity so the transport is visible
        F = F * (1.0 + 0.1 * np.random.default_rng(9).random(F.shape[:dxd]))[(...,) + (None,) * dv]
    ghosts = workloads.ghost_vectors(c)
    solid = workloads.solid_mask(c)
    ctx = fks.Context(dv, dxd, M, N, L, A, h=c["dx"], bc=c["bc"])
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    if solid is not None:
        ctx.set_solid(solid)
    ctx.set_params(tau=c["tau"])
    fin = dev(torch, F)
    out = torch.empty_like(fin)
    ctx.step(fin, out, c["dt"])
    ctx.check()
    got = host(out).reshape((-1,) + (N,) * dv)
    tab = tables.build_tables(dv, N, L)
    fstar = transport.gather(F, 0, dxd, dv, N, L, c["dt"], c["dx"], c["bc"], ghosts, cells=sample)
    flatF = F.reshape((-1,) + (N,) * dv)
    for i, cell in enumerate(sample):
        if solid is not None and solid.reshape(-1)[cell]:
            np.testing.assert_array_equal(got[cell], flatF[cell])
            continue
        Q = oproj.project_zero_moments(collision.collide_fft(fstar[i], tab), dv, N, L)
        ref = fstar[i] + (c["dt"] / c["tau"]) * Q
        assert np.max(np.abs(got[cell] - ref)) <= TOL * np.max(np.abs(ref)), (name, cell)


@pytest.mark.parametrize("scheme", [None, "heun_strang"])
def test_in_place_calls_bitwise(torch, fks, scheme):
    """§8(b) in-place calls (f_out == f_in: the north_star's fks_step(f, dt)): collide, transport,
    step and step_bgk on one buffer equal the out-of-place calls bitwise (1D x 3D, ghost / outflow
    faces, a solid cell; the default scheme and Heun + Strang)."""
    N, L, M = 8, 7.0, [6]
    bc = [transport.GHOST, transport.OUTFLOW]
    h = 0.1
    dt = 0.9 * h / (L - L / N)
    F = workloads.family("smooth", 3, N, L, 6, seed=17) * np.linspace(0.6, 1.4, 6)[:, None, None, None]
    g = workloads.family("smooth", 3, N, L, 1, seed=18)[0]
    solid = np.array([0, 0, 1, 0, 0, 0], dtype=bool)
    ctxs = []
    for _ in range(2):
        c = fks.Context(3, 1, M, N, L, 24, h=h, bc=bc)
        c.set_ghost(0, dev(torch, g))
        c.set_solid(solid)
        if scheme:
            c.set_scheme(fks.SPLIT_STRANG, fks.TIME_HEUN)
        ctxs.append(c)
    a = dev(torch, F)
    b = torch.empty_like(a)
    ctxs[0].collide(a, b)
    x = a.clone()
    ctxs[1].collide(x, x)
    assert torch.equal(x, b)
    calls = [lambda c, i, o: c.step(i, o, dt), lambda c, i, o: c.transport(i, o, dt)]
    if not scheme:
        calls.append(lambda c, i, o: c.step_bgk(i, o, dt, bgk.NU_RHO, 0.0))
    x = a.clone()
    for call in calls:
        b = torch.empty_like(a)
        call(ctxs[0], a, b)
        call(ctxs[1], x, x)
        assert torch.equal(x, b)
        a = b
    for c in ctxs:
        c.check()
