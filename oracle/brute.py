"""Brute-force quadrature of the Boltzmann operator in its sigma-representation (oracle; tests only).

P:129-137 (eq. bolt): Q_B(f)(v) = int_{R^d} int_{S^{d-1}} B(|v - v*|, omega)
    [f(v') f(v'*) - f(v) f(v*)] d omega d v*,
    v' = (v + v* + |q| omega)/2,  v'* = (v + v* - |q| omega)/2  (reading #11: the printed v'*
    has a sign typo), q = v - v*.
P:141-157: B = |q| sigma; Maxwell molecules (2D here): B = b0; VHS hard spheres (3D): B = C1 |q|.

This evaluates the integral directly, for an analytic f given as a callable, by a trapezoid
rule in v* on a wide box and a product rule in omega (uniform on S^1; Gauss-Legendre in
cos(theta) x uniform phi on S^2).  It shares nothing with the spectral evaluators: it pins
the spectral operator as a whole -- constants, psi reading, truncation radius.
"""
import numpy as np


def _omega_2d(K):
    th = 2.0 * np.pi * np.arange(K) / K
    return np.stack([np.cos(th), np.sin(th)], axis=1), np.full(K, 2.0 * np.pi / K)


def _omega_3d(Kt, Kp):
    x, wx = np.polynomial.legendre.leggauss(Kt)  # cos(theta) nodes on [-1, 1]
    ph = 2.0 * np.pi * np.arange(Kp) / Kp
    C, P = np.meshgrid(x, ph, indexing="ij")
    S = np.sqrt(1.0 - C * C)
    om = np.stack([S * np.cos(P), S * np.sin(P), C], axis=-1).reshape(-1, 3)
    w = (wx[:, None] * np.full(Kp, 2.0 * np.pi / Kp)[None, :]).reshape(-1)
    return om, w


def boltzmann_Q(fun, v, d, kernel, W=8.0, h=0.1, K=64, Kt=24, Kp=48, split=False):
    """Q_B(f)(v) at one point v (length d).  kernel: 'maxwell2d' (B = 1/(2 pi)) or
    'hs3d' (B = |q| / (4 pi)).  Returns Q (or (gain, loss) if split)."""
    g1 = np.arange(-W, W + 0.5 * h, h)
    wts1 = np.full(g1.shape, h)
    wts1[0] = wts1[-1] = 0.5 * h
    mesh = np.meshgrid(*([g1] * d), indexing="ij")
    vstar = np.stack([m.reshape(-1) for m in mesh], axis=1)  # [M, d]
    wv = np.ones(1)
    for _ in range(d):
        wv = np.multiply.outer(wv, wts1)
    wv = wv.reshape(-1)
    v = np.asarray(v, dtype=np.float64)
    q = v[None, :] - vstar
    qn = np.linalg.norm(q, axis=1)
    if kernel == "maxwell2d":
        B = np.full(qn.shape, 1.0 / (2.0 * np.pi))
        om, wo = _omega_2d(K)
    elif kernel == "hs3d":
        B = qn / (4.0 * np.pi)
        om, wo = _omega_3d(Kt, Kp)
    else:
        raise ValueError(kernel)
    fv = fun(v[None, :])[0]
    fstar = fun(vstar)
    loss = fv * np.sum(wv * B * fstar) * np.sum(wo)
    center = 0.5 * (v[None, :] + vstar)            # [M, d]
    gain = 0.0
    for o, w in zip(om, wo):
        half = 0.5 * qn[:, None] * o[None, :]
        gain += w * np.sum(wv * B * fun(center + half) * fun(center - half))
    if split:
        return gain, loss
    return gain - loss


def gaussian_mixture(centers, temps, masses):
    """f(v) = sum_i m_i (2 pi T_i)^{-d/2} exp(-|v - c_i|^2 / (2 T_i)) as a callable on [..., d]."""
    centers = np.atleast_2d(np.asarray(centers, dtype=np.float64))
    d = centers.shape[1]

    def fun(x):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros(x.shape[:-1])
        for c, T, m in zip(centers, temps, masses):
            r2 = np.sum((x - c) ** 2, axis=-1)
            out += m * (2.0 * np.pi * T) ** (-d / 2.0) * np.exp(-r2 / (2.0 * T))
        return out
    return fun
