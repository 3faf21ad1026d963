"""Pins of the NEXT-3 oracle (general decoupled kernels, reading #25) against things other
than itself: closed forms of phi_{R,a}, arbitrary-precision quadrature,
Fresnel integrals, exact polynomial integration of the Gauss-Jacobi rule, the closed-form loss
frequencies of the decoupled kernel, and a brute-force evaluation of the paper's Carleman integral
 that uses no Fourier transform.  None of these touch the CUDA path.
"""
import mpmath
import numpy as np
import pytest
from scipy.special import fresnel

from oracle import brute, collision, grid, kernels, moments, tables

R = 2.8


@pytest.mark.parametrize("gamma", [-0.5, 0.0, 0.5, 1.0, 1.7, 2.0])
def test_gauss_jacobi_integrates_polynomials_exactly(gamma):
    """int_0^1 t^gamma t^k dt = 1 / (gamma + k + 1) for k <= 2n - 1 (the defining property)."""
    n = 40
    t, w = kernels.gauss_jacobi01(n, gamma)
    assert np.all((t > 0) & (t < 1)) and np.all(w > 0)
    for k in (0, 1, 7, 30, 79):
        assert abs(np.sum(w * t ** k) * (gamma + k + 1.0) - 1.0) <= 5e-14


@pytest.mark.parametrize("s", [0.0, 0.3, 2.9, 13.0, 55.0])
def test_phi_a_closed_forms(s):
    """gamma = 0: phi2 = 2 R sinc(R s); gamma = 1: phi3; gamma = 2:
    2 [(R^2 s^2 - 2) sin(R s) + 2 R s cos(R s)] / s^3 (elementary antiderivative);
    gamma = -1/2: 2 sqrt(R) sqrt(2 pi / z) C(sqrt(2 z / pi)), z = R s (Fresnel C)."""
    scale = 2 * R ** 3
    assert abs(kernels.phi_a(s, R, 0.0) - kernels.phi2(s, R)) <= 1e-14 * scale
    assert abs(kernels.phi_a(s, R, 1.0) - kernels.phi3(s, R)) <= 1e-14 * scale
    if s == 0.0:
        g2 = 2 * R ** 3 / 3
        gm = 4 * np.sqrt(R)
    else:
        g2 = 2 * ((R * R * s * s - 2) * np.sin(R * s) + 2 * R * s * np.cos(R * s)) / s ** 3
        z = R * s
        gm = 2 * np.sqrt(R) * np.sqrt(2 * np.pi / z) * fresnel(np.sqrt(2 * z / np.pi))[1]
    assert abs(kernels.phi_a(s, R, 2.0) - g2) <= 1e-14 * scale
    assert abs(kernels.phi_a(s, R, -0.5) - gm) <= 1e-14 * 4 * np.sqrt(R)


@pytest.mark.parametrize("gamma", [0.5, 1.7, -0.3])
def test_phi_a_vs_arbitrary_precision(gamma):
    """phi_{R,a}(s) = int_{-R}^{R} |rho|^gamma e^{i rho s} d rho by mpmath tanh-sinh at 30 digits."""
    mpmath.mp.dps = 30
    for s in (0.0, 0.7, 9.0, 31.0):
        ref = 2 * mpmath.quad(lambda r: r ** gamma * mpmath.cos(r * s), mpmath.linspace(0, R, 12))
        assert abs(kernels.phi_a(s, R, gamma) - float(ref)) <= 2e-14 * float(2 * R ** (gamma + 1))


def _maxwellian3(N, L, u, T, rho):
    vs = grid.velocity_components(3, N, L)
    f = rho * np.exp(-((vs[0] - u) ** 2 + vs[1] ** 2 + vs[2] ** 2) / (2 * T)) / (2 * np.pi * T) ** 1.5
    return vs, f


@pytest.mark.parametrize("gamma,tol", [(0.0, 1e-5), (2.0, 1e-4)])
def test_loss_frequency_3d_decoupled(gamma, tol):
    """Loss of the decoupled kernel (reading #25): int int Btilde delta(x.y) F(x+y) dx dy =
    4 C (2 pi / (gamma+1)) int |q|^gamma F(q) dq, so for a Maxwellian
    gamma = 0 (3D Maxwell molecules): Q^- = 8 pi C rho f (constant frequency);
    gamma = 2: Q^- = (8 pi C / 3) rho (|v-u|^2 + 3T) f.  Pins the unit scaling kappa^{-(3+gamma)},
    the quadrature of phi_{R,a} and the 2 pi/(gamma+1) angular factor."""
    N, L = 32, 8.0
    u, T, rho = 0.3, 1.0, 1.0
    vs, f = _maxwellian3(N, L, u, T, rho)
    C = 1.0 / (4 * np.pi)
    tab = tables.build_tables(3, N, L, gamma=gamma)
    _, _, l = collision.collide_fft(f, tab, return_parts=True)
    r2 = (vs[0] - u) ** 2 + vs[1] ** 2 + vs[2] ** 2
    nu = 8 * np.pi * C * rho * (np.ones_like(f) if gamma == 0.0 else (r2 + 3 * T) / 3)
    bulk = np.sqrt(vs[0] ** 2 + vs[1] ** 2 + vs[2] ** 2) < 2.5
    assert np.max(np.abs(l[bulk] / f[bulk] / nu[bulk] - 1)) < tol


def test_loss_frequency_2d_gamma2():
    """2D, gamma = 2: int_{cos>0} cos^2 = pi/2, so Q^- = 2 C (pi/2) rho (|v-u|^2 + 2T) f."""
    N, L = 32, 9.0
    vx, vy = grid.velocity_components(2, N, L)
    f = 1.3 * np.exp(-((vx - 0.3) ** 2 + vy ** 2) / 1.6) / (2 * np.pi * 0.8)
    tab = tables.build_tables(2, N, L, A=8, gamma=2.0)
    _, _, l = collision.collide_fft(f, tab, return_parts=True)
    rho = moments.moments(f, 2, N, L)[0]
    nu = 2 * (1 / (2 * np.pi)) * (np.pi / 2) * rho * ((vx - 0.3) ** 2 + vy ** 2 + 2 * 0.8)
    mask = np.sqrt(vx ** 2 + vy ** 2) < 3
    assert np.max(np.abs(l[mask] / f[mask] / nu[mask] - 1)) < 1e-4


@pytest.mark.parametrize("gamma", [0.0, 1.0, 2.0, 0.5])
def test_brute_force_carleman_2d(gamma):
    """The spectral operator with decoupled tables (N = 64, A = 16) equals the brute-force
    Carleman integral (no FFT) to 1e-9 of max|Q^-|: constants, scaling and phi_{R,a} together."""
    fun = brute.gaussian_mixture([[-0.8, 0.3], [0.7, -0.2]], [0.4, 0.5], [0.6, 0.5])
    N, L = 64, 8.0
    vx, vy = grid.velocity_components(2, N, L)
    pts = np.stack([vx, vy], -1)
    tab = tables.build_tables(2, N, L, A=16, gamma=gamma)
    Q, g, l = collision.collide_fft(fun(pts), tab, return_parts=True)
    scale = np.max(np.abs(l))
    for (i, j) in [(N // 2, N // 2), (N // 2 + 5, N // 2 + 5), (N // 2 - 4, N // 2 + 1)]:
        qb = brute.carleman_Q(fun, pts[i, j], 2, gamma, 1 / (2 * np.pi), tab.R * L / np.pi)
        assert abs(qb - Q[i, j]) <= 1e-9 * scale


@pytest.mark.parametrize("gamma", [0.0, 2.0, 0.5])
def test_brute_force_carleman_3d(gamma):
    """3D, N = 32: the 24-design operator is within 1e-2 of max|Q^-| of the brute-force Carleman
    integral (its angular quadrature error), and with the (theta, phi) product grid the gain error
    falls like A^-2 from 8x8 to 12x12 directions (second-order midpoint rule): the decoupled
    tables converge to the paper's integral, not to something else."""
    fun = brute.gaussian_mixture([[-0.6, -0.4, -0.2], [0.6, 0.4, 0.2]], [0.6, 0.6], [0.5, 0.5])
    N, L = 32, 8.0
    pts = np.stack(grid.velocity_components(3, N, L), -1)
    idx = (17, 15, 18)
    Ru = tables.default_R() * L / np.pi
    gb, lb = brute.carleman_Q(fun, pts[idx], 3, gamma, 1 / (4 * np.pi), Ru, split=True)
    tab = tables.build_tables(3, N, L, gamma=gamma)
    Q, g, l = collision.collide_fft(fun(pts), tab, return_parts=True)
    assert abs((gb - lb) - Q[idx]) <= 1e-2 * np.max(np.abs(l))
    if gamma != 2.0:
        return
    errs = []
    for A1 in (8, 12):
        t = tables.build_tables(3, N, L, gamma=gamma, directions=kernels.directions_3d_product(A1, A1))
        _, gA, _ = collision.collide_fft(fun(pts), t, return_parts=True)
        errs.append(abs(gA[idx] - gb) / gb)
    assert errs[0] < 5e-3 and errs[1] < errs[0] / 1.8      # (12/8)^2 = 2.25


def test_decoupled_operator_conserves_mass_and_is_bilinear():
    """The general-gamma tables keep the structural invariants of P5/P15: Qhat_0 = 0 (mass) and
    Q(2f) = 4 Q(f)."""
    N, L = 16, 7.0
    tab = tables.build_tables(3, N, L, gamma=0.5)
    f = np.random.default_rng(3).random((N,) * 3) * _maxwellian3(N, L, 0.0, 3.0, 1.0)[1]
    Q = collision.collide_fft(f, tab)
    _, g, l = collision.collide_fft(f, tab, return_parts=True)
    assert abs(Q.sum()) <= 1e-14 * np.abs(l).sum()
    assert np.max(np.abs(collision.collide_fft(2 * f, tab) - 4 * Q)) <= 1e-14 * np.max(np.abs(g) + np.abs(l)) * 4
