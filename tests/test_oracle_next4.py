"""Pins of the NEXT-4 oracle (reading #26): the Heun (RK2) collision integrator
 and Strang splitting with FKS half-step transports, against things other
than themselves -- the BKW exact solution and Table 1, the convergence order of the
integrator, exact composition of the half-step gathers with the full-step gather and with the
exact particle positions, conservation, and the accuracy gain over the paper's first-order scheme.
"""
import os

import numpy as np

import workloads
from oracle import bkw, grid, projection, step, tables, transport


def _bkw_start(N, L):
    vx, vy = grid.velocity_components(2, N, L)
    v2 = vx ** 2 + vy ** 2
    return v2, projection.project_to_moments(bkw.bkw_initial(v2), [1.0, 0.0, 0.0, 2.0], 2, N, L)


def test_heun_is_second_order_euler_first():
    """Self-convergence of the 0D collision ODE (BKW start, N = 16): halving dt divides the
    successive differences by 4 for Heun and by 2 for forward Euler."""
    N, L = 16, 6.0
    tab = tables.build_tables(2, N, L, A=8)
    _, f0 = _bkw_start(N, L)
    for integ, order in (("euler", 1), ("heun", 2)):
        res = []
        for k in (10, 20, 40, 80):
            f = f0.copy()
            for _ in range(k):
                f = step.homogeneous_step(f[None], tab, 1.0 / k, integrator=integ)[0]
            res.append(f)
        e = [np.abs(res[i] - res[i + 1]).max() for i in range(3)]
        for i in range(2):
            assert abs(e[i] / e[i + 1] - 2 ** order) < 0.15 * 2 ** order


def test_heun_bkw_below_table1(golden_dir):
    """BKW exact solution at t = 10, N = 32, the printed Delta t = 0.02: Heun
    reaches the spectral floor -- at least 10x below Table 1's N = 32 L1 error, and
    halving dt no longer changes the error by more than 20%."""
    rows = {}
    for line in open(os.path.join(golden_dir, "table1_bkw.txt")):
        if line.strip() and not line.startswith("#"):
            n_, L_, l1, l2 = line.split()
            rows[int(n_)] = (float(L_), float(l1))
    N = 32
    L, l1_paper = rows[N]
    tab = tables.build_tables(2, N, L, A=8)
    v2, f0 = _bkw_start(N, L)
    fe = bkw.bkw(v2, 10.0)
    errs = []
    for dt in (0.02, 0.01):
        f = f0.copy()
        for _ in range(int(round(10.0 / dt))):
            f = step.homogeneous_step(f[None], tab, dt, integrator="heun")[0]
        errs.append(np.abs(f - fe).sum() / np.abs(fe).sum())
    assert errs[0] < l1_paper / 10
    assert abs(errs[0] / errs[1] - 1) < 0.2


def test_half_step_shifts_compose_to_the_full_step():
    """Strang's half transports (positions p dt/2) are the paper's FKS shift sampled twice as often:
    s_half(2n) = s(n) bitwise; sum over the two half steps = the full-step delta; and two periodic
    half-step gathers equal one full-step gather bitwise (the transport is exact)."""
    N, L, dx = 8, 3.0, 0.25
    bc = [transport.PERIODIC] * 4
    rng = np.random.default_rng(7)
    for cfl in (0.9, 1.7):
        dt = cfl * dx / (L - L / N)
        for n in range(40):
            np.testing.assert_array_equal(transport.shift_s_half(2 * n, N, L, dt, dx), transport.shift_s(n, N, L, dt, dx))
            np.testing.assert_array_equal(
                transport.shift_delta_half(2 * n, N, L, dt, dx) + transport.shift_delta_half(2 * n + 1, N, L, dt, dx),
                transport.shift_delta(n, N, L, dt, dx))
        F = rng.random((5, 7, N, N))
        for n in (0, 3, 11):
            full = transport.gather(F, n, 2, 2, N, L, dt, dx, bc)
            h1 = transport.gather(F, n, 2, 2, N, L, dt, dx, bc, delta=transport.shift_delta_half(2 * n, N, L, dt, dx))
            h2 = transport.gather(h1, n, 2, 2, N, L, dt, dx, bc, delta=transport.shift_delta_half(2 * n + 1, N, L, dt, dx))
            np.testing.assert_array_equal(h2, full)


def test_half_step_positions_are_exact():
    """After p half steps the value at x_j is the initial piece containing x_j - p v dt / 2 (exact
    positions, computed here without the shift formula)."""
    N, L, M, dx = 8, 3.0, 11, 0.25
    dt = 0.0731
    F0 = np.random.default_rng(8).random((M, N, N))
    F = F0.copy()
    bc = [transport.PERIODIC] * 2
    for p in range(25):
        F = transport.gather(F, 0, 1, 2, N, L, dt, dx, bc, delta=transport.shift_delta_half(p, N, L, dt, dx))
    v = grid.nodes_1d(N, L)
    for kx in range(N):
        for j in range(M):
            xj = (j + 0.5) * dx - 25 * v[kx] * dt / 2
            src = int(np.floor(xj / dx)) % M
            np.testing.assert_array_equal(F[j, :, kx], F0[src, :, kx])


def _smooth_1d(N, L, M):
    vs = grid.velocity_components(2, N, L)
    x = (np.arange(M) + 0.5) / M
    return np.stack([workloads.gen.maxwellian(vs, 1 + 0.3 * np.sin(2 * np.pi * xi), (0.3 * np.cos(2 * np.pi * xi), 0.0),
                                              1.0 + 0.2 * np.sin(2 * np.pi * xi)) for xi in x])


def _run(F0, tab, N, L, M, dt, tf, integ, split):
    cfg = dict(dx_dim=1, dv=2, N=N, L=L, dt=dt, dx=1.0 / M, tau=0.05, bc=[0, 0])
    F = F0.copy()
    for n in range(int(round(tf / dt))):
        F = step.step(F, n, cfg, tab, integrator=integ, splitting=split)
    return F


def test_strang_and_heun_conserve_and_reduce_the_time_error():
    """1D x 2D periodic smooth flow (tau = 0.05, t = 0.1): every scheme conserves mass exactly;
    against a fine Strang + Heun reference, Strang splitting beats the paper's Lie + Euler scheme
     at the same dt, and Strang + Heun beats it by more."""
    N, L, M, tf = 8, 4.0, 16, 0.1
    tab = tables.build_tables(2, N, L, A=8)
    F0 = _smooth_1d(N, L, M)
    ref = _run(F0, tab, N, L, M, tf / 320, tf, "heun", "strang")
    assert abs(ref.sum() / F0.sum() - 1) < 1e-13
    for k in (10, 20):
        e = {}
        for integ, split in (("euler", "lie"), ("euler", "strang"), ("heun", "strang")):
            F = _run(F0, tab, N, L, M, tf / k, tf, integ, split)
            assert abs(F.sum() / F0.sum() - 1) < 1e-13
            e[(integ, split)] = np.abs(F - ref).max() / np.abs(ref).max()
        assert e[("euler", "strang")] < e[("euler", "lie")] / 1.5
        assert e[("heun", "strang")] < e[("euler", "lie")] / 3


def test_strang_equals_lie_without_spatial_variation():
    """A spatially uniform periodic state: every transport is the identity, so Strang = Lie bitwise."""
    N, L, M = 8, 4.0, 6
    vs = grid.velocity_components(2, N, L)
    m = workloads.gen.maxwellian(vs, 1.0, (0.4, -0.2), 0.9) * (1 + 0.01 * np.random.default_rng(2).random((N, N)))
    F = np.broadcast_to(m, (M, N, N)).copy()
    tab = tables.build_tables(2, N, L, A=8)
    for integ in ("euler", "heun"):
        cfg = dict(dx_dim=1, dv=2, N=N, L=L, dt=0.03, dx=0.1, tau=0.5, bc=[0, 0])
        a = step.step(F, 3, cfg, tab, integrator=integ, splitting="lie")
        b = step.step(F, 3, cfg, tab, integrator=integ, splitting="strang")
        np.testing.assert_array_equal(a, b)
