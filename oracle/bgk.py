"""BGK relaxation with the conservative (projected) Maxwellian — NEXT-2 (oracle; test infrastructure only).

P:122-127 (eq. ibgk): Q_BGK(f) = nu (M[f] - f), nu > 0 the collision frequency.
P:909: the rescaled equation d_t f + v.grad f = Q(f) / tau.
P:944: nu = rho (Maxwellian molecules comparisons); nu = mu, a constant.
P:359-364 (eq. minimMax): the discrete Maxwellian is the pointwise equilibrium E~[f] = M(v_k)
corrected onto the moments U = C f of the cell, E[U] = E~ + C^T (C C^T)^{-1} (U - C E~), so mass,
momentum and energy are conserved exactly on the lattice (C = Delta v^d Phi; the factor cancels).
P:259-275 (eq. f_coll): forward Euler, f^{n+1} = f* + (dt / tau) nu (E[f*] - f*).
Euler limit (tau -> 0, "the limit model of compressible Euler equations"): f^{n+1} = E[f*].

Maxwellian (reading #12): M(v) = rho / (2 pi T)^{d/2} exp(-|v - u|^2 / (2 T)) with
(rho, u, T) the moments of f (oracle/moments.py); nodes are cell centred (reading #14).
"""
import numpy as np

from . import grid, moments, projection

NU_RHO, NU_CONST, NU_EULER = 0, 1, 2


def maxwellian(rho, u, T, d, N, L):
    """Pointwise Maxwellian at the velocity nodes, shape (N,)*d."""
    vs = grid.velocity_components(d, N, L)
    r2 = sum((v - u[a]) ** 2 for a, v in enumerate(vs))
    return rho / (2.0 * np.pi * T) ** (d / 2.0) * np.exp(-r2 / (2.0 * T))


def conservative_maxwellian(f, d, N, L):
    """E[U(f)] of eq. minimMax: the Maxwellian of f's moments, projected onto them."""
    rho, u, T = moments.moments(f, d, N, L)
    Et = maxwellian(rho, u, T, d, N, L)
    Phi = projection.moment_rows(d, N, L)
    U = Phi @ f.reshape(-1)  # the Delta v^d factor of C cancels in eq. minimMax
    lam = np.linalg.solve(Phi @ Phi.T, U - Phi @ Et.reshape(-1))
    return (Et.reshape(-1) + Phi.T @ lam).reshape(f.shape)


def bgk_step_cell(f, dt, tau, nu_rule, mu, d, N, L):
    """One forward-Euler BGK step of one cell (or the Euler limit)."""
    E = conservative_maxwellian(f, d, N, L)
    if nu_rule == NU_EULER:
        return E
    nu = moments.moments(f, d, N, L)[0] if nu_rule == NU_RHO else mu
    return f + (dt / tau) * nu * (E - f)


def homogeneous_bgk_step(fs, dt, tau, nu_rule, mu, d, N, L):
    return np.stack([bgk_step_cell(f, dt, tau, nu_rule, mu, d, N, L) for f in fs])
