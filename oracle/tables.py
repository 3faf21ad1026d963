"""Spectral quadrature tables alpha_p, alpha'_p and the loss symbol D (oracle; tests only).

P:446-452: beta_F(l, m) ~= sum_p alpha_p(l) alpha'_p(m) turns Q into A convolutions.
2D: B_F(l, m) = (pi/A) sum_p phi^2(l . e_p) phi^2(m . e_p^perp).
3D: B_F(l, m) = sum_p w_p phi^3(l . e_p) psi^3(|Pi_{e_p^perp}(m)|),
                |Pi_{e^perp}(m)| computed as |m x e| (no cancellation).
P:438: beta_F(l, m) = B_F(l, m) - B_F(m, m); the loss symbol is
       D(m) = B_F(m, m) / Btilde = sum_p w_p alpha_p(m) alpha'_p(m).

Reading #10 (Nyquist): alpha and alpha' are symmetrised over the index reflection
sigma, alpha <- (alpha + alpha o sigma) / 2, before D is formed, so every table is even on
the lattice and F^{-1}[alpha f^] is real for real f.

Reading #3/#7 (constants): Btilde = 2^{d-1} B |q|^{-(d-2)} with B the collision kernel
(not sigma): 2D Maxwell molecules B = b0 -> Btilde = 2 b0; 3D hard spheres B = C1 |q| ->
Btilde = 4 C1.  Defaults b0 = 1/(2 pi), C1 = 1/(4 pi) (so Btilde = 1/pi in both).
App. A.1 of SURVEY (unit scaling): Q_user = kappa^{-(d+gamma)} Q_scaled, kappa = pi / L.
The overall node-space factor is s = Btilde * kappa^{-(d+gamma)}.
"""
from dataclasses import dataclass

import numpy as np

from . import grid, kernels

LAMBDA = 2.0 / (3.0 + np.sqrt(2.0))


@dataclass
class Tables:
    d: int
    N: int
    L: float
    R: float
    gamma: float
    alpha: np.ndarray   # [A, (N,)*d]
    alphap: np.ndarray  # [A, (N,)*d]
    D: np.ndarray       # [(N,)*d]
    w: np.ndarray       # [A]
    scale: float        # s = Btilde * kappa^-(d+gamma)

    @property
    def A(self):
        return self.w.shape[0]


def default_R():
    """Reading #1: default truncation radius 2 lambda pi (scaled units)."""
    return 2.0 * LAMBDA * np.pi


def build_tables(d, N, L, directions=None, A=8, R=None, kernel_const=None, psi="derived",
                 symmetrise=True, gamma=None):
    """Build the tables for d=2 (Maxwell molecules, gamma=0) or d=3 (hard spheres, gamma=1).

    directions: for d=2 the number A of angles is used; for d=3 a tuple (e, w) of
    unit vectors [A,3] and weights [A] (default: the 24-point design, reading #17).
    gamma (NEXT-3, reading #25): VHS exponent of B = C |q|^gamma; at gamma = d - 2 the
    Carleman kernel is constant and the tables are the closed forms above; any other
    gamma > -1 uses the decoupled model Btilde(x, y) = 2^{d-1} C |x|^{gamma-(d-2)} (b = 1), i.e.
    alpha_p = phi_{R,a}(l . e_p) by quadrature (kernels.phi_a) and alpha'_p
    unchanged (phi2 in 2D, psi3 in 3D).
    """
    if R is None:
        R = default_R()
    kappa = np.pi / L
    ls = grid.mode_vectors(d, N)
    if d == 2:
        gamma = 0.0 if gamma is None else float(gamma)
        b0 = 1.0 / (2.0 * np.pi) if kernel_const is None else kernel_const
        Btilde = 2.0 * b0
        e, ep, w = kernels.directions_2d(A)
        rad = (lambda s: kernels.phi2(s, R)) if gamma == 0.0 else (lambda s: kernels.phi_a(s, R, gamma))
        alpha = np.stack([rad(ls[0] * e[p, 0] + ls[1] * e[p, 1]) for p in range(len(w))])
        alphap = np.stack([kernels.phi2(ls[0] * ep[p, 0] + ls[1] * ep[p, 1], R) for p in range(len(w))])
    elif d == 3:
        gamma = 1.0 if gamma is None else float(gamma)
        C1 = 1.0 / (4.0 * np.pi) if kernel_const is None else kernel_const
        Btilde = 4.0 * C1
        if directions is None:
            e, w = kernels.directions_3d_design24()
        else:
            e, w = directions
        psif = kernels.psi3 if psi == "derived" else kernels.psi3_printed
        al, alp = [], []
        for p in range(len(w)):
            ex, ey, ez = e[p]
            dot = ls[0] * ex + ls[1] * ey + ls[2] * ez
            cx = ls[1] * ez - ls[2] * ey
            cy = ls[2] * ex - ls[0] * ez
            cz = ls[0] * ey - ls[1] * ex
            perp = np.sqrt(cx * cx + cy * cy + cz * cz)
            al.append(kernels.phi3(dot, R) if gamma == 1.0 else kernels.phi_a(dot, R, gamma))
            alp.append(psif(perp, R))
        alpha, alphap = np.stack(al), np.stack(alp)
    else:
        raise ValueError("d must be 2 or 3")
    if symmetrise:
        alpha = 0.5 * (alpha + np.stack([grid.mirror(a) for a in alpha]))
        alphap = 0.5 * (alphap + np.stack([grid.mirror(a) for a in alphap]))
    D = np.einsum("p,p...->...", w, alpha * alphap)
    scale = Btilde * kappa ** (-(d + gamma))
    return Tables(d=d, N=N, L=L, R=R, gamma=gamma, alpha=alpha, alphap=alphap, D=D, w=np.asarray(w),
                  scale=scale)
