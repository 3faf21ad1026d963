"""Radial functions and quadrature direction sets (oracle; test infrastructure only).

All in the paper's scaled velocity units (box [-pi, pi]^d).

2D Maxwell molecules:  phi_R^2(s) = int_{-R}^{R} e^{i rho s} d rho = 2 R sinc(R s).
3D hard spheres:       phi_R^3(s) = R^2 [2 sinc(R s) - sinc^2(R s / 2)]
                                  (= int_{-R}^{R} |rho| e^{i rho s} d rho, reading #4).
psi_R^3: the paper prints 2 R^2 sinc^2(R s / 2) but its own derivation (P:501-506,
"integrating first e' on the intersection of the unit sphere with the plane e^perp") gives
the great-circle integral int_0^pi phi_R^3(s cos theta) d theta = 2 pi R J_1(R s) / s,
psi(0) = pi R^2 (reading #2).  ``psi3`` is the derived form; ``psi3_printed`` is kept for the
pins that discriminate the two (P8/P9).

Directions:
  2D (reading #5): theta_p = pi p / A, p = 1..A, e_p = (cos, sin),
      e_p^perp = e_{theta_p + pi/2}, weight pi / A.
  3D product grid (reading #6): theta_p = (p + 1/2) pi / A1, phi_q = q pi / A2,
      e = (sin th cos ph, sin th sin ph, cos th), weight pi^2 sin(theta_p) / (A1 A2),
      renormalised so that sum w = 2 pi (the measure of the half sphere S^2_+).
  3D 24-point spherical 7-design (reading #17): orbit of the chiral octahedral group O
      (the 24 signed permutation matrices with det +1) of a point p whose squared
      coordinates a < b < c are the roots of 105 t^3 - 105 t^2 + 21 t - 1 = 0, i.e.
      a+b+c = 1, ab+bc+ca = 1/5, abc = 1/105 -- the conditions that make every
      O-invariant harmonic of degree 4 and 6 vanish at p (odd degrees vanish by the
      group), so the orbit integrates all polynomials of degree <= 7 exactly.
      Weight 2 pi / 24 (half-sphere measure, integrands are even).
"""
import itertools

import numpy as np
from scipy.special import j1


def sinc(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.ones_like(x)
    nz = x != 0.0
    out[nz] = np.sin(x[nz]) / x[nz]
    return out


def phi2(s, R):
    """phi_R^2(s) = 2 R sinc(R s)."""
    return 2.0 * R * sinc(R * np.asarray(s, dtype=np.float64))


def phi3(s, R):
    """phi_R^3(s) = R^2 [2 sinc(R s) - sinc^2(R s / 2)]."""
    s = np.asarray(s, dtype=np.float64)
    return R * R * (2.0 * sinc(R * s) - sinc(0.5 * R * s) ** 2)


def psi3(s, R):
    """psi_R^3(s) = 2 pi R J1(R s) / s, psi(0) = pi R^2  (derived reading #2 of P:501-519)."""
    s = np.asarray(s, dtype=np.float64)
    out = np.full_like(s, np.pi * R * R)
    nz = s != 0.0
    out[nz] = 2.0 * np.pi * R * j1(R * s[nz]) / s[nz]
    return out


def psi3_printed(s, R):
    """The formula as printed at P:525: 2 R^2 sinc^2(R s / 2) (kept for pins only)."""
    s = np.asarray(s, dtype=np.float64)
    return 2.0 * R * R * sinc(0.5 * R * s) ** 2


# ---------------------------------------------------------------- NEXT-3: general decoupled kernels
def gauss_jacobi01(n, gamma):
    """Nodes t_i, weights w_i with sum_i w_i g(t_i) = int_0^1 t^gamma g(t) dt exactly for polynomials
    g of degree <= 2n-1 (gamma > -1).  Golub-Welsch: the nodes are the eigenvalues of the Jacobi
    matrix of the Jacobi polynomials P^(0, gamma) on [-1, 1] (numpy eigvalsh as the library
    primitive), polished by Newton on the orthonormal three-term recurrence; the weights come from
    the Christoffel sum w_i = 1 / sum_{k<n} q_k(x_i)^2 (accurate to a few ulp); t = (1 + x) / 2."""
    a, b = 0.0, float(gamma)
    k = np.arange(n, dtype=np.float64)
    ab = a + b
    alpha = np.empty(n)
    alpha[0] = (b - a) / (ab + 2.0)
    kk = k[1:]
    alpha[1:] = (b * b - a * a) / ((2 * kk + ab) * (2 * kk + ab + 2.0))
    kk = np.arange(1, n + 1, dtype=np.float64)   # beta_1 .. beta_n
    beta = 4.0 * kk * (kk + a) * (kk + b) * (kk + ab) / ((2 * kk + ab) ** 2 * (2 * kk + ab + 1.0) * (2 * kk + ab - 1.0))
    sb = np.sqrt(beta)
    from scipy.special import gammaln
    mu0 = np.exp((ab + 1.0) * np.log(2.0) + gammaln(a + 1.0) + gammaln(b + 1.0) - gammaln(ab + 2.0))
    J = np.diag(alpha) + np.diag(sb[:-1], 1) + np.diag(sb[:-1], -1)
    x = np.sort(np.linalg.eigvalsh(J))

    def recur(x):
        """q_0..q_n and q_n' at the points x (orthonormal recurrence)."""
        qm, q = np.zeros_like(x), np.full_like(x, 1.0 / np.sqrt(mu0))
        dm, dq = np.zeros_like(x), np.zeros_like(x)
        ssum = q * q
        for j in range(n):
            qn = ((x - alpha[j]) * q - (sb[j - 1] if j else 0.0) * qm) / sb[j]
            dn = (q + (x - alpha[j]) * dq - (sb[j - 1] if j else 0.0) * dm) / sb[j]
            qm, q, dm, dq = q, qn, dq, dn
            if j < n - 1:
                ssum = ssum + q * q
        return q, dq, ssum

    for _ in range(3):
        qn, dqn, _ = recur(x)
        x = x - qn / dqn
    _, _, ssum = recur(x)
    w = 1.0 / ssum
    return 0.5 * (1.0 + x), w * 2.0 ** (-b - 1.0)


def phi_a(s, R, gamma, nodes=160):
    """NEXT-3 (P:498-509, P:537-538 with reading #4): phi_{R,a}(s) = int_{-R}^{R} |rho|^gamma e^{i rho s}
    d rho = 2 R^{gamma+1} int_0^1 t^gamma cos(R s t) dt, the radial factor of the decoupled kernel
    Btilde(x, y) = 2^{d-1} C |x|^{gamma-(d-2)} b(|y|), b = 1 (d = 3: |rho| a(|rho|) with
    a = |rho|^{gamma-1}; d = 2: a(|rho|) = |rho|^gamma).  gamma = 1 (d = 3) gives phi3, gamma = 0
    gives phi2.  Evaluated by Gauss-Jacobi quadrature with the t^gamma weight (gamma > -1)."""
    s = np.asarray(s, dtype=np.float64)
    t, w = gauss_jacobi01(nodes, gamma)
    z = (R * s).reshape(-1)
    out = np.empty(z.shape)
    for c0 in range(0, z.size, 65536):
        zz = z[c0:c0 + 65536]
        out[c0:c0 + 65536] = np.cos(np.multiply.outer(zz, t)) @ w
    return (2.0 * R ** (gamma + 1.0) * out).reshape(s.shape)


def directions_2d(A):
    """(e [A,2], e_perp [A,2], w [A]) with theta_p = pi p / A, p = 1..A, w = pi/A."""
    th = np.pi * np.arange(1, A + 1) / A
    e = np.stack([np.cos(th), np.sin(th)], axis=1)
    ep = np.stack([-np.sin(th), np.cos(th)], axis=1)
    w = np.full(A, np.pi / A)
    return e, ep, w


def directions_3d_product(A1, A2, renormalise=True):
    """Midpoint-in-theta product grid on the half sphere (reading #6)."""
    th = (np.arange(A1) + 0.5) * np.pi / A1
    ph = np.arange(A2) * np.pi / A2
    T, P = np.meshgrid(th, ph, indexing="ij")
    e = np.stack([np.sin(T) * np.cos(P), np.sin(T) * np.sin(P), np.cos(T)], axis=-1).reshape(-1, 3)
    w = (np.pi ** 2 * np.sin(T) / (A1 * A2)).reshape(-1)
    if renormalise:
        w = w * (2.0 * np.pi / w.sum())
    return e, w


def octahedral_rotations():
    """The 24 signed permutation matrices with determinant +1 (chiral octahedral group O),
    in a fixed order: permutations in lexicographic order, then sign patterns."""
    mats = []
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((1.0, -1.0), repeat=3):
            M = np.zeros((3, 3))
            for r in range(3):
                M[r, perm[r]] = signs[r]
            if np.linalg.det(M) > 0:
                mats.append(M)
    assert len(mats) == 24
    return mats


def design_24_generator():
    """p = (sqrt a, sqrt b, sqrt c), a < b < c roots of 105 t^3 - 105 t^2 + 21 t - 1."""
    roots = np.sort(np.roots([105.0, -105.0, 21.0, -1.0]).real)
    # polish each root by Newton on the cubic (np.roots is an eigenvalue solve)
    for _ in range(3):
        p = 105 * roots ** 3 - 105 * roots ** 2 + 21 * roots - 1
        dp = 315 * roots ** 2 - 210 * roots + 21
        roots = roots - p / dp
    return np.sqrt(roots)


def directions_3d_design24():
    """24-point spherical 7-design, w = 2 pi / 24 (reading #17)."""
    p = design_24_generator()
    e = np.array([M @ p for M in octahedral_rotations()])
    w = np.full(24, 2.0 * np.pi / 24)
    return e, w
