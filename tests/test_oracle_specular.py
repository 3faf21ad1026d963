"""Pins of the specular-reflection transport (NEXT-1, oracle/transport.gather_specular), CPU only.

Fixed by closed properties rather than by the oracle itself: without solids it is the plain
gather (P12-pinned); in a closed (periodic) box the gather is a permutation of fluid values, so
mass and energy over the fluid cells are conserved exactly; a Maxwellian at rest is invariant
(even in every velocity component); a single particle hitting a wall comes back with the normal
velocity component negated.
"""
import numpy as np
import pytest

import workloads
from oracle import grid, transport


def _case(M, dv, N, L, seed):
    rng = np.random.default_rng(seed)
    shape = tuple(M[::-1]) + (N,) * dv
    return rng.uniform(0.1, 1.0, shape)


@pytest.mark.parametrize("dxd,dv,M,N", [(1, 2, [7], 8), (2, 2, [5, 4], 8), (2, 3, [4, 3], 8)])
def test_no_solids_equals_plain_gather(dxd, dv, M, N):
    L, dx = 5.0, 0.1
    dt = 0.9 * dx / (L - L / N)
    bc = [transport.GHOST, transport.OUTFLOW] + [transport.PERIODIC] * (2 * dxd - 2)
    F = _case(M, dv, N, L, 1)
    ghosts = {0: workloads.family("smooth", dv, N, L, 1, seed=3)[0]}
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    for n in range(3):
        a = transport.gather(F, n, dxd, dv, N, L, dt, dx, bc, ghosts)
        b = transport.gather_specular(F, n, dxd, dv, N, L, dt, dx, bc, ghosts, solid)
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("dxd,dv,M,N,blocks", [(1, 2, [9], 8, [(4,)]), (2, 2, [6, 5], 8, [(2, 2), (3, 2)]),
                                               (2, 2, [6, 6], 8, [(2, 2), (3, 2), (2, 3)]),  # L shape
                                               (2, 3, [5, 4], 8, [(1, 2)]),
                                               (3, 3, [4, 4, 3], 8, [(1, 1, 1), (2, 1, 1), (1, 2, 1)])])
def test_closed_box_conserves_mass_and_energy(dxd, dv, M, N, blocks):
    """Periodic box with interior solid cells: the gather permutes the fluid values."""
    L, dx = 5.0, 0.1
    dt = 0.95 * dx / (L - L / N)
    bc = [transport.PERIODIC] * (2 * dxd)
    F = _case(M, dv, N, L, 2)
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    for b in blocks:
        solid[tuple(reversed(b))] = True
    fluid = ~solid
    v2 = sum(v * v for v in grid.velocity_components(dv, N, L))
    for n in range(4):
        G = transport.gather_specular(F, n, dxd, dv, N, L, dt, dx, bc, None, solid)
        assert np.array_equal(np.sort(F[fluid].reshape(-1)), np.sort(G[fluid].reshape(-1)))
        assert abs(np.sum(G[fluid] * v2) - np.sum(F[fluid] * v2)) <= 1e-12 * np.sum(F[fluid] * v2)
        np.testing.assert_array_equal(G[solid], F[solid])
        F = G


def test_maxwellian_at_rest_is_invariant():
    dxd, dv, M, N, L, dx = 2, 2, [6, 5], 16, 6.0, 0.1
    dt = 0.9 * dx / (L - L / N)
    vs = grid.velocity_components(dv, N, L)
    Mx = np.exp(-sum(v * v for v in vs) / 2)
    F = np.broadcast_to(Mx, tuple(M[::-1]) + Mx.shape).copy()
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    solid[2, 3] = solid[2, 4] = True
    for n in range(3):
        G = transport.gather_specular(F, n, dxd, dv, N, L, dt, dx, [transport.PERIODIC] * 4, None, solid)
        np.testing.assert_array_equal(G, F)


def test_single_particle_reflects_off_a_wall():
    """1D x 2D: a particle in cell 3 moving +x toward the solid cell 4 comes back with v_x negated."""
    dxd, dv, M, N, L, dx = 1, 2, [8], 8, 4.0, 0.1
    vmax = L - L / N
    dt = 0.9 * dx / vmax
    solid = np.zeros((8,), dtype=bool)
    solid[4] = True
    kx, ky = N - 1, 2                      # largest +v_x: shifts every step at CFL 0.9
    F = np.zeros((8, N, N))
    F[3, ky, kx] = 1.0                     # layout [cell][ky][kx]
    delta = transport.shift_delta(0, N, L, dt, dx)
    assert delta[kx] == -1                 # the source of +v_x is the cell below: this one moves up
    G = transport.gather_specular(F, 0, dxd, dv, N, L, dt, dx, [transport.PERIODIC] * 2, None, solid)
    assert G[3, ky, N - 1 - kx] == 1.0 and np.sum(G) == 1.0


def test_reentry_inflow_schedule():
    """eq. BCs: the printed branches, |u_BC| = 3 throughout, continuity at t1, t2."""
    f = workloads.reentry_inflow_velocity
    t1, t2 = 1.5, 3 * np.sqrt(2) / 2 + 1.5
    assert f(1.0) == (3.0, 0.0)
    assert np.allclose(f(t2 + 0.5), (3 * np.sqrt(2) / 2, 3 * np.sqrt(2) / 2), rtol=0, atol=1e-15)
    assert np.allclose(f(t1 + 1.0), (2 * np.sqrt(2), 1.0), rtol=0, atol=1e-15)
    for t in np.linspace(0, 10, 101):
        assert abs(np.hypot(*f(t)) - 3.0) < 1e-14
    for tj in (t1, t2):
        assert np.allclose(f(tj - 1e-12), f(tj + 1e-12), atol=1e-9)
