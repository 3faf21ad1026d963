"""BKW exact solution of the 2D Maxwell-molecule Boltzmann equation (oracle; tests only).

P:733-747: f(v, 0) = |v|^2/pi exp(-|v|^2);
f(v, t) = 1/(2 pi S^2) exp(-|v|^2/(2S)) [2S - 1 + (1-S)/(2S) |v|^2],  S = 1 - exp(-t/8)/2.
"""
import numpy as np


def S(t):
    return 1.0 - 0.5 * np.exp(-t / 8.0)


def bkw(v2, t):
    """Exact BKW density at |v|^2 = v2 and time t."""
    s = S(t)
    return np.exp(-v2 / (2.0 * s)) / (2.0 * np.pi * s * s) * (2.0 * s - 1.0 + (1.0 - s) / (2.0 * s) * v2)


def bkw_initial(v2):
    """P:734."""
    return v2 / np.pi * np.exp(-v2)
