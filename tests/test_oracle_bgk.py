"""Pins of the BGK oracle (NEXT-2) against closed forms and invariants (CPU only).

Each pin fixes a part of oracle/bgk.py by something other than the oracle itself: the
analytic moments of a Gaussian (normalisation, sign of the exponent, the factor 2 in 2T),
the exact conservation identities of eq. minimMax, the fixed point of the projected
Maxwellian, the forward-Euler algebra of eq. f_coll, and the monotone relaxation of BGK.
"""
import numpy as np
import pytest

import workloads
from oracle import bgk, grid, moments, projection


@pytest.mark.parametrize("d,N,L", [(2, 32, 8.0), (3, 32, 8.0)])
def test_maxwellian_moments_closed_form(d, N, L):
    """A well-resolved Gaussian on a wide cell-centred grid has its analytic moments (the
    midpoint rule is spectrally accurate for it): pins the normalisation rho/(2 pi T)^(d/2),
    the -|v-u|^2/(2T) exponent and the velocity offset."""
    rho, u, T = 1.3, np.array([0.4, -0.3, 0.2][:d]), 0.9
    M = bgk.maxwellian(rho, u, T, d, N, L)
    r, uu, TT = moments.moments(M, d, N, L)
    assert abs(r - rho) < 1e-10 * rho
    assert np.max(np.abs(uu - u)) < 1e-10
    assert abs(TT - T) < 1e-10
    # and the exact peak value at a node placed on u = 0
    M0 = bgk.maxwellian(1.0, np.zeros(d), 1.0, d, N, L)
    v = grid.nodes_1d(N, L)
    k = N // 2
    assert np.isclose(M0[(k,) * d], (2 * np.pi) ** (-d / 2) * np.exp(-d * v[k] ** 2 / 2), rtol=1e-15)


@pytest.mark.parametrize("d,N,L,kind", [(2, 32, 9.0, "random"), (2, 16, 6.0, "smooth"), (3, 16, 7.0, "random")])
def test_conservative_maxwellian_has_the_moments_of_f(d, N, L, kind):
    """eq. minimMax: C E[U] = U exactly (to rounding), whatever f is."""
    f = workloads.family(kind, d, N, L, 3, seed=5)
    Phi = projection.moment_rows(d, N, L)
    for c in range(3):
        E = bgk.conservative_maxwellian(f[c], d, N, L)
        a, b = Phi @ f[c].reshape(-1), Phi @ E.reshape(-1)
        assert np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300)) < 1e-12


def test_conservative_maxwellian_fixed_point():
    """E depends on f only through its moments, and has them: E[E[f]] = E[f]."""
    d, N, L = 2, 32, 9.0
    f = workloads.family("random", d, N, L, 1, seed=8)[0]
    E = bgk.conservative_maxwellian(f, d, N, L)
    E2 = bgk.conservative_maxwellian(E, d, N, L)
    assert np.max(np.abs(E2 - E)) <= 1e-13 * np.max(np.abs(E))


def test_conservative_maxwellian_of_a_maxwellian():
    """For a resolved Maxwellian the correction of eq. minimMax is tiny: E[M] = M (closed form)."""
    d, N, L = 3, 32, 8.0
    M = bgk.maxwellian(0.8, np.array([0.3, 0.0, -0.2]), 1.1, d, N, L)
    E = bgk.conservative_maxwellian(M, d, N, L)
    assert np.max(np.abs(E - M)) <= 1e-9 * np.max(M)


@pytest.mark.parametrize("nu_rule,mu", [(bgk.NU_RHO, 0.0), (bgk.NU_CONST, 2.5)])
def test_bgk_step_algebra_and_conservation(nu_rule, mu):
    d, N, L = 2, 32, 9.0
    f = workloads.family("random", d, N, L, 2, seed=11)
    tau = 0.7
    Phi = projection.moment_rows(d, N, L)
    for c in range(2):
        rho = moments.moments(f[c], d, N, L)[0]
        nu = rho if nu_rule == bgk.NU_RHO else mu
        # (dt / tau) nu = 1: one step lands exactly on E (eq. f_coll algebra)
        dt = tau / nu
        E = bgk.conservative_maxwellian(f[c], d, N, L)
        g = bgk.bgk_step_cell(f[c], dt, tau, nu_rule, mu, d, N, L)
        assert np.max(np.abs(g - E)) <= 1e-14 * np.max(np.abs(E))
        # a fractional step conserves the moments and halves the distance at (dt/tau) nu = 1/2
        g = bgk.bgk_step_cell(f[c], 0.5 * dt, tau, nu_rule, mu, d, N, L)
        a, b = Phi @ f[c].reshape(-1), Phi @ g.reshape(-1)
        assert np.max(np.abs(a - b) / np.abs(a)) < 1e-12
        assert np.max(np.abs((g - E) - 0.5 * (f[c] - E))) <= 1e-14 * np.max(np.abs(f[c]))
    # Euler limit: the equilibrium itself
    g = bgk.bgk_step_cell(f[0], 0.1, tau, bgk.NU_EULER, 0.0, d, N, L)
    np.testing.assert_array_equal(g, bgk.conservative_maxwellian(f[0], d, N, L))


def test_bgk_relaxation_monotone():
    """||f^n - E||_2 is non-increasing under (dt/tau) nu < 1 (the moments, hence E, are invariant)."""
    d, N, L = 2, 32, 9.0
    f = workloads.family("smooth", d, N, L, 1, seed=2)[0]
    E = bgk.conservative_maxwellian(f, d, N, L)
    prev = np.linalg.norm(f - E)
    for _ in range(6):
        f = bgk.bgk_step_cell(f, 0.3, 1.0, bgk.NU_CONST, 1.0, d, N, L)
        cur = np.linalg.norm(f - E)
        assert cur <= prev * (1 + 1e-12)
        prev = cur
