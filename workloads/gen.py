"""Synthetic workloads shaped like the paper's tests.

Seeds: numpy PCG64(160808009 + config_id).  Node coordinates follow the cell-centred reading
v_k = -L + (k + 1/2) 2L/N; arrays are [cells..., k_z, k_y, k_x] fp64 (x fastest).

C1  0Dx2D BKW ensemble, Maxwell molecules, N=32, L=9, A=8          (Test 1.1)
C2  0Dx3D two-Gaussian relaxation ensemble, hard spheres, N=32, L=7 (Test 1.3)
C3  1Dx3D Sod, Nx=400 on [0,2], N=32, L=16, tau=1e-2              (Test 2.3)
C4  2Dx3D re-entry geometry, 100^2 on [0,4]^2, N=32, L=10          (Test 3.2 geometry P:1491-1504)
C5  3Dx3D re-entry, 48^3 on [0,2]^3, N=32, L=10, tau=0.3           (Test 4.1)
"""
import numpy as np

PERIODIC, GHOST, OUTFLOW = 0, 1, 2

CONFIGS = {
    "C1": dict(cid=1, dx_dim=0, dv=2, N=32, L=9.0, A=8, cells=(65536,), dt=0.02, tau=1.0, steps=10),
    "C2": dict(cid=2, dx_dim=0, dv=3, N=32, L=7.0, A=24, cells=(4096,), dt=0.05, tau=1.0, steps=10),
    "C3": dict(cid=3, dx_dim=1, dv=3, N=32, L=16.0, A=24, cells=(400,), extent=2.0, tau=1e-2, steps=20,
               bc=[GHOST, GHOST]),
    "C4": dict(cid=4, dx_dim=2, dv=3, N=32, L=10.0, A=24, cells=(100, 100), extent=4.0, tau=1e-2, steps=10,
               bc=[GHOST, OUTFLOW, OUTFLOW, OUTFLOW]),
    "C5": dict(cid=5, dx_dim=3, dv=3, N=32, L=10.0, A=24, cells=(48, 48, 48), extent=2.0, tau=0.3, steps=5,
               bc=[GHOST, OUTFLOW, OUTFLOW, OUTFLOW, OUTFLOW, OUTFLOW]),
}


def _nodes(N, L):
    return -L + (np.arange(N) + 0.5) * (2.0 * L / N)


def _vgrid(dv, N, L):
    v1 = _nodes(N, L)
    g = np.meshgrid(*([v1] * dv), indexing="ij")
    return [g[dv - 1 - a] for a in range(dv)]  # component a (0 = x) in [k_z, k_y, k_x] layout


def config(name, **over):
    """Config dict; spatial configs get dx = extent / M and the CFL-1 dt = dx / max|v_k|_inf
    (reading #15)."""
    c = dict(CONFIGS[name])
    c.update(over)
    c["name"] = name
    if c["dx_dim"] > 0:
        c["dx"] = c["extent"] / c["cells"][-1]
        vmax = c["L"] - c["L"] / c["N"]
        c.setdefault("dt", c["dx"] / vmax)
    return c


def maxwellian(vs, rho, u, T):
    d = len(vs)
    r2 = sum((v - ui) ** 2 for v, ui in zip(vs, u))
    return rho * np.exp(-r2 / (2.0 * T)) / (2.0 * np.pi * T) ** (d / 2.0)


def _rng(c, salt=0):
    return np.random.Generator(np.random.PCG64(160808009 + c["cid"] + 1000 * salt))


def initial_state(c, ncells=None, start=0):
    """Initial f for the config (optionally only cells [start, start+ncells) of the flat cell
    list, for the 0D ensembles)."""
    dv, N, L = c["dv"], c["N"], c["L"]
    vs = _vgrid(dv, N, L)
    name = c["name"]
    if name == "C1":
        tot = c["cells"][0]
        rng = _rng(c)
        rho = rng.uniform(0.5, 1.5, tot)
        u = rng.uniform(-0.5, 0.5, (tot, 2))
        n = tot if ncells is None else ncells
        out = np.empty((n, N, N))
        for i in range(n):
            k = start + i
            r2 = (vs[0] - u[k, 0]) ** 2 + (vs[1] - u[k, 1]) ** 2
            out[i] = rho[k] * r2 / np.pi * np.exp(-r2)          # P:734 shifted/scaled
        return out
    if name == "C2":
        tot = c["cells"][0]
        rng = _rng(c)
        rho = rng.uniform(0.5, 1.5, tot)
        q = rng.standard_normal((tot, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        v1 = np.array([-1.0, -1.0, -0.25])
        s2 = 0.2
        n = tot if ncells is None else ncells
        out = np.empty((n, N, N, N))
        for i in range(n):
            k = start + i
            a, b, cc, d = q[k]
            Rm = np.array([[1 - 2 * (cc * cc + d * d), 2 * (b * cc - a * d), 2 * (b * d + a * cc)],
                           [2 * (b * cc + a * d), 1 - 2 * (b * b + d * d), 2 * (cc * d - a * b)],
                           [2 * (b * d - a * cc), 2 * (cc * d + a * b), 1 - 2 * (b * b + cc * cc)]])
            w = Rm @ v1
            g1 = np.exp(-sum((v - wi) ** 2 for v, wi in zip(vs, w)) / (2 * s2))
            g2 = np.exp(-sum((v + wi) ** 2 for v, wi in zip(vs, w)) / (2 * s2))
            out[i] = rho[k] * (g1 + g2) / (2.0 * (2 * np.pi * s2) ** 1.5)
        return out
    M = c["cells"]  # (M_{dx-1}, ..., M_0)
    if name == "C3":
        left = maxwellian(vs, 1.0, (0, 0, 0), 2.5)
        right = maxwellian(vs, 0.125, (0, 0, 0), 0.25)
        x = (np.arange(M[0]) + 0.5) * c["dx"]
        return np.stack([left if xi <= 1.0 else right for xi in x])
    if name in ("C4", "C5"):
        u = (3.0, 0.0, 0.0) if name == "C4" else (2.0, 0.0, 0.0)
        m = maxwellian(vs, 1.0, u, 1.0)
        lead = tuple(M) if ncells is None else (ncells,)   # ncells: that many (flat) cells only
        return np.broadcast_to(m, lead + m.shape).copy()
    raise KeyError(name)


def ghost_vectors(c):
    """{face: ghost vector} for the GHOST faces (Dirichlet/inflow, frozen, reading #19)."""
    dv, N, L = c["dv"], c["N"], c["L"]
    vs = _vgrid(dv, N, L)
    if c["name"] == "C3":
        return {0: maxwellian(vs, 1.0, (0, 0, 0), 2.5), 1: maxwellian(vs, 0.125, (0, 0, 0), 0.25)}
    if c["name"] == "C4":
        return {0: maxwellian(vs, 1.0, (3.0, 0.0, 0.0), 1.0)}   # eq. BCs first phase
    if c["name"] == "C5":
        return {0: maxwellian(vs, 1.0, (2.0, 0.0, 0.0), 1.0)}
    return {}


def reentry_inflow_velocity(t):
    """(u_x, u_y)_BC(t) of eq. BCs: (3, 0) up to t1 = 3/2, then (sqrt(9 - g^2), g) with
    g = t - t1 up to t2 = 3 sqrt(2)/2 + t1, then (3 sqrt(2)/2, 3 sqrt(2)/2): a speed-3 inflow turning
    by 45 degrees (NEXT-1 "time-dependent inflow schedule")."""
    t1 = 1.5
    t2 = 3.0 * np.sqrt(2.0) / 2.0 + t1
    if t <= t1:
        return (3.0, 0.0)
    if t <= t2:
        g = t - t1
        return (float(np.sqrt(9.0 - g * g)), float(g))
    return (3.0 * np.sqrt(2.0) / 2.0, 3.0 * np.sqrt(2.0) / 2.0)


def reentry_inflow_ghost(c, t):
    """The west-face inflow ghost vector of C4 at time t: Maxwellian (rho, T) = (1, 1) with the
    velocity of eq. BCs (boundary data, pointwise like the initial data)."""
    dv, N, L = c["dv"], c["N"], c["L"]
    ux, uy = reentry_inflow_velocity(t)
    return maxwellian(_vgrid(dv, N, L), 1.0, (ux, uy, 0.0)[:dv], 1.0)


def solid_mask(c):
    """Boolean [cells...] of solid cells (cell centre inside an obstacle), or None."""
    if c["name"] == "C4":
        M = c["cells"]
        h = c["dx"]
        x = (np.arange(M[1]) + 0.5) * h
        y = (np.arange(M[0]) + 0.5) * h
        Y, X = np.meshgrid(y, x, indexing="ij")
        x0, x1, xp0, xp1 = 1.5, 1.7, 1.8, 2.0
        y0, y1, yp0, yp1 = 1.7, 1.95, 2.05, 2.3
        box = lambda a, b, c_, d: (X >= a) & (X <= b) & (Y >= c_) & (Y <= d)  # noqa: E731
        return box(x0, x1, y0, y1) | box(x0, x1, yp0, yp1) | box(xp0, xp1, (y0 + yp0) / 2, (y1 + yp1) / 2)
    if c["name"] == "C5":
        M = c["cells"]
        h = c["dx"]
        x = (np.arange(M[0]) + 0.5) * h
        Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
        inside = lambda a: (a >= 0.75) & (a <= 1.25)  # noqa: E731   reading #19
        return inside(X) & inside(Y) & inside(Z)
    return None


def family(kind, dv, N, L, ncells, seed=0):
    """Parity input families: 'smooth' (random Maxwellian per cell),
    'neareq' (Maxwellian x (1 + 1e-6 noise)), 'random' (U[0,1) x Gaussian envelope, stresses
    Nyquist handling), 'bkw' (2D only)."""
    rng = np.random.Generator(np.random.PCG64(160808009 + 77 * seed + 13 * dv + N))
    vs = _vgrid(dv, N, L)
    out = np.empty((ncells,) + (N,) * dv)
    for i in range(ncells):
        rho = rng.uniform(0.5, 1.5)
        u = rng.uniform(-0.15, 0.15, dv) * L
        T = rng.uniform(0.04, 0.08) * L * L
        m = maxwellian(vs, rho, u, T)
        if kind == "smooth":
            out[i] = m
        elif kind == "neareq":
            out[i] = m * (1.0 + 1e-6 * rng.standard_normal(m.shape))
        elif kind == "random":
            env = maxwellian(vs, 1.0, np.zeros(dv), 0.08 * L * L)
            out[i] = rng.random(m.shape) * env
        elif kind == "bkw" and dv == 2:
            r2 = (vs[0] - u[0] / L) ** 2 + (vs[1] - u[1] / L) ** 2
            out[i] = rho * r2 / np.pi * np.exp(-r2)
        else:
            raise ValueError(kind)
    return out


class ScaledField:
    """Lazy stand-in for a [cells..., (N,)*dv] array F[j] = s[j] * v (one fp64 product per element,
    exactly what a device-side broadcast multiply computes), for full-size parity tests whose state
    does not fit the host's numpy comfortably.  Supports .shape and the tuple indexing the oracle's
    gathers use (spatial indices first, then velocity indices; integers or broadcastable arrays)."""

    def __init__(self, v, s):
        self.v = np.asarray(v, dtype=np.float64)
        self.s = np.asarray(s, dtype=np.float64)
        self.shape = self.s.shape + self.v.shape

    def __getitem__(self, idx):
        if not isinstance(idx, tuple):
            idx = (idx,)
        ns = self.s.ndim
        sp, vel = idx[:ns], idx[ns:]
        vel = vel + (slice(None),) * (self.v.ndim - len(vel))
        return self.s[sp] * self.v[vel]
