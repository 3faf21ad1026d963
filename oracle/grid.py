"""Velocity lattice and Fourier-mode bookkeeping (oracle; test infrastructure only).

P:179-191 -- "a cubic grid in velocity space of N points with Delta v the grid
step which is taken equal in each direction".  Reading #14: nodes are
cell-centred, v_k = -L + (k + 1/2) Delta v.  Array layout: a cell's
distribution is an ndarray of shape (N,)*d indexed [k_z, k_y, k_x] (x fastest);
``velocity_components`` returns the user-unit velocity component arrays in the
same layout, component 0 = v_x.

P:379-389 -- truncated Fourier series on [-pi, pi]^d (after the scaling
kappa = pi / L, reading #1).  Modes are stored in FFT wrap order: index j <-> mode
mu(j) = j for j < N/2, j - N otherwise (reading #9).
"""
import numpy as np


def nodes_1d(N, L):
    """Cell-centred nodes of one velocity axis, v_k = -L + (k + 1/2) * (2L/N)."""
    dv = 2.0 * L / N
    return -L + (np.arange(N) + 0.5) * dv


def spacing(N, L):
    return 2.0 * L / N


def velocity_components(d, N, L):
    """List [v_x, v_y(, v_z)] of arrays of shape (N,)*d (index order [k_z,k_y,k_x])."""
    v1 = nodes_1d(N, L)
    grids = np.meshgrid(*([v1] * d), indexing="ij")  # grids[a] varies along array axis a
    # array axis 0 is the slowest (z in 3D, y in 2D); component x is the last axis
    return [grids[d - 1 - a] for a in range(d)]


def mode_numbers_1d(N):
    """mu(j): FFT wrap order mode numbers in [-N/2, N/2)."""
    j = np.arange(N)
    return np.where(j < N // 2, j, j - N)


def mode_vectors(d, N):
    """List [l_x, l_y(, l_z)] of integer mode arrays of shape (N,)*d (same layout as f)."""
    m1 = mode_numbers_1d(N)
    grids = np.meshgrid(*([m1] * d), indexing="ij")
    return [grids[d - 1 - a].astype(np.float64) for a in range(d)]


def mirror(arr):
    """arr o sigma, sigma(l)_a = mu((-j_a) mod N): the index-space reflection l -> -l
    (Nyquist index N/2 maps to itself)."""
    out = arr
    for ax in range(arr.ndim):
        out = np.roll(np.flip(out, axis=ax), 1, axis=ax)
    return out
