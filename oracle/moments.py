"""Macroscopic moments (oracle; test infrastructure only).

P:96-113: U = int f phi(v) dv, phi = (1, v, |v|^2); Maxwellian with (1/2) d rho T = E - (1/2) rho |u|^2.
Reading #12: T = int |v - u|^2 f dv / (d rho) (the printed E carries a factor 1/2 ambiguity;
T is unambiguous).  Discrete version (eq. DM): sums times Delta v^d.
"""
import numpy as np

from . import grid


def moments(f, d, N, L):
    """(rho, u[d], T) of one cell's node values f (shape (N,)*d)."""
    dv = grid.spacing(N, L) ** d
    vs = grid.velocity_components(d, N, L)
    rho = dv * np.sum(f)
    u = np.array([dv * np.sum(v * f) / rho for v in vs])
    e = dv * np.sum(sum(v * v for v in vs) * f) / rho
    T = (e - np.dot(u, u)) / d
    return rho, u, T


def moments_batch(fs, d, N, L):
    out = [moments(f, d, N, L) for f in fs]
    return (np.array([o[0] for o in out]), np.array([o[1] for o in out]), np.array([o[2] for o in out]))
