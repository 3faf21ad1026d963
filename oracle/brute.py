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


def carleman_Q(fun, v, d, gamma, C, R, nr=40, Kt=16, Kp=32, Ky=32, split=False):
    """NEXT-3: Q(f)(v) straight from the paper's Carleman form (eq. defQBCarleman)
    Q(v) = int int Btilde(x, y) delta(x . y) [f(v + y) f(v + x) - f(v + x + y) f(v)] dx dy
    with the decoupled model Btilde(x, y) = 2^{d-1} C |x|^{gamma-(d-2)} (b = 1; reading #25)
    and the spectral method's truncation |x|, |y| <= R (user units: R = R_scaled L / pi).

    No Fourier anything: x = rho e (rho in [0, R] by Gauss-Jacobi with the rho^gamma weight that
    remains after the Jacobian rho^{d-1} and delta(x . y) = delta(e . y) / rho; e over the whole
    sphere: Gauss-Legendre in cos(theta) x uniform phi in 3D, uniform on S^1 in 2D), y over the
    disk (3D, polar: r Gauss-Legendre x uniform angle) or the segment (2D) of radius R in e^perp."""
    from .kernels import gauss_jacobi01
    v = np.asarray(v, dtype=np.float64)
    K = 2.0 ** (d - 1) * C
    t, wt = gauss_jacobi01(nr, gamma)
    rho, wrho = R * t, wt * R ** (gamma + 1.0)          # int_0^R rho^gamma g = sum wrho g(rho)
    fv = fun(v[None, :])[0]
    if d == 3:
        es, we = _omega_3d(Kt, Kp)
        xr, wr = np.polynomial.legendre.leggauss(nr)     # r in [0, R], weight r dr
        r = 0.5 * R * (xr + 1.0)
        wr = 0.5 * R * wr * r
        ph = 2.0 * np.pi * np.arange(Ky) / Ky
        gain = loss = 0.0
        for e, w_e in zip(es, we):
            a = np.array([1.0, 0.0, 0.0]) if abs(e[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
            e1 = np.cross(e, a)
            e1 /= np.linalg.norm(e1)
            e2 = np.cross(e, e1)
            ys = (r[:, None, None] * (np.cos(ph)[None, :, None] * e1 + np.sin(ph)[None, :, None] * e2)).reshape(-1, 3)
            wy = np.repeat(wr, Ky) * (2.0 * np.pi / Ky)
            xs = rho[:, None] * e[None, :]                             # [nr, 3]
            fy = fun(v[None, :] + ys)                                   # [ny]
            fx = fun(v[None, :] + xs)                                   # [nr]
            fxy = fun(v[None, None, :] + xs[:, None, :] + ys[None, :, :])  # [nr, ny]
            gain += w_e * np.sum(wrho * fx * (fy @ wy))
            loss += w_e * fv * np.sum(wrho * (fxy @ wy))
    elif d == 2:
        th = 2.0 * np.pi * np.arange(Kt * Kp) / (Kt * Kp)
        xl, wl = np.polynomial.legendre.leggauss(2 * nr)            # y = s e_perp, s in [-R, R]
        sy, wy = R * xl, R * wl
        gain = loss = 0.0
        for a in th:
            e = np.array([np.cos(a), np.sin(a)])
            ep = np.array([-np.sin(a), np.cos(a)])
            ys = sy[:, None] * ep[None, :]
            xs = rho[:, None] * e[None, :]
            fy = fun(v[None, :] + ys)
            fx = fun(v[None, :] + xs)
            fxy = fun(v[None, None, :] + xs[:, None, :] + ys[None, :, :])
            w_e = 2.0 * np.pi / (Kt * Kp)
            gain += w_e * np.sum(wrho * fx * (fy @ wy))
            loss += w_e * fv * np.sum(wrho * (fxy @ wy))
    else:
        raise ValueError(d)
    gain, loss = K * gain, K * loss
    if split:
        return gain, loss
    return gain - loss
