"""L2 conservation projection (oracle; test infrastructure only).

P:319-358: given f~ and the moment matrix C = Delta v^d [1; v_k; |v_k|^2], the
minimiser of ||f~ - f||_2 subject to C f = U is f = f~ + C^T (C C^T)^{-1} (U - C f~) (eq. minim1,
P:355-356).  Reading #13: the collision output is projected onto zero moments,
Pi Q = Q - Phi^T (Phi Phi^T)^{-1} Phi Q with Phi = C / Delta v^d (the factor cancels), which
is algebraically identical to projecting f~ = f* + dt Q onto U = C f* (SURVEY App. A.8).
"""
import numpy as np

from . import grid


def moment_rows(d, N, L):
    """Phi [(d+2), n]: rows 1, v_x, .., v_{d-1}, |v|^2 at the nodes (flat layout of f)."""
    vs = grid.velocity_components(d, N, L)
    rows = [np.ones(N ** d)] + [v.reshape(-1) for v in vs] + [sum(v * v for v in vs).reshape(-1)]
    return np.array(rows)


def project_zero_moments(Q, d, N, L):
    """Pi Q (P:355-356 with U = 0)."""
    Phi = moment_rows(d, N, L)
    q = Q.reshape(-1)
    lam = np.linalg.solve(Phi @ Phi.T, Phi @ q)
    return (q - Phi.T @ lam).reshape(Q.shape)


def project_to_moments(f, U, d, N, L):
    """f + C^T (C C^T)^{-1} (U - C f) with C = Delta v^d Phi; U = (rho, rho u, int |v|^2 f)."""
    Phi = moment_rows(d, N, L) * grid.spacing(N, L) ** d
    x = f.reshape(-1)
    lam = np.linalg.solve(Phi @ Phi.T, np.asarray(U, dtype=np.float64) - Phi @ x)
    return (x + Phi.T @ lam).reshape(f.shape)
