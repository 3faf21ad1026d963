"""One split step (oracle; test infrastructure only).

P:226-233: Lie splitting, transport first then collision.
P:259-275 (eq. f_coll): forward Euler on the cell-centred values, f^{n+1} = f* + dt Q(f*).
P:909: the rescaled equation d_t f + v.grad f = Q(f)/tau.
P:319-320 + reading #13: the collision output is projected to zero moments.
Solid cells (reading #19) keep their values; the collision is skipped there.

NEXT-4 ("many different time integrators can be employed", "time accuracy
can be increased by high order time splitting methods"; reading #26):
  integrator "heun": the explicit second-order Runge-Kutta (Heun) step of the collision ODE
      f1 = f* + (dt/tau) PiQ(f*),  f^{n+1} = f* + (dt/2tau) [PiQ(f*) + PiQ(f1)];
  splitting "strang": f^{n+1} = T(dt/2) C(dt) T(dt/2) f^n, each half transport an FKS gather
      between the half-step positions 2n -> 2n+1 -> 2n+2 (transport.shift_delta_half).
"""
import numpy as np

from . import collision, projection, transport


def _transport(F, n, cfg, delta=None):
    dxd, dv, N, L = cfg["dx_dim"], cfg["dv"], cfg["N"], cfg["L"]
    if cfg.get("specular"):
        return transport.gather_specular(F, n, dxd, dv, N, L, cfg["dt"], cfg.get("dx", 1.0), cfg.get("bc"),
                                         cfg.get("ghosts") or {}, cfg["solid"], delta=delta)
    out = transport.gather(F, n, dxd, dv, N, L, cfg["dt"], cfg.get("dx", 1.0), cfg.get("bc"), cfg.get("ghosts"),
                           delta=delta)
    solid = cfg.get("solid")
    if solid is not None:               # reading #19: solid cells keep their values
        out[solid] = F[solid]
    return out


def _collision_update(fj, cfg, tab, coll, integrator):
    """Euler or Heun (NEXT-4) for one cell's collision ODE, projected Q (reading #13)."""
    dv, N, L = cfg["dv"], cfg["N"], cfg["L"]
    h = cfg["dt"] / cfg["tau"]

    def pq(g):
        Q = coll(g, tab)
        return projection.project_zero_moments(Q, dv, N, L) if cfg.get("project", True) else Q
    Q1 = pq(fj)
    if integrator == "euler":
        return fj + h * Q1
    f1 = fj + h * Q1
    return fj + (0.5 * h) * (Q1 + pq(f1))


def _collide_all(Fs, F, cfg, tab, evaluator, integrator):
    dxd = cfg["dx_dim"]
    coll = collision.collide_fft if evaluator == "fft" else collision.collide_direct
    sp_shape = F.shape[:dxd]
    solid = cfg.get("solid")
    out = np.empty_like(F)
    for jflat in range(int(np.prod(sp_shape)) if dxd else 1):
        jidx = np.unravel_index(jflat, sp_shape) if dxd else ()
        if solid is not None and solid[jidx]:
            out[jidx] = F[jidx]          # reading #19: solid cells keep their values
            continue
        out[jidx] = _collision_update(Fs[jidx], cfg, tab, coll, integrator)
    return out


def step(F, n, cfg, tab, evaluator="fft", integrator="euler", splitting="lie"):
    """F^{n+1} from F^n.  cfg: dict with dx_dim, dv, N, L, dt, dx, tau, bc, ghosts, solid, project
    (and specular).  integrator: "euler" | "heun"; splitting: "lie" | "strang" (NEXT-4)."""
    dxd, N, L = cfg["dx_dim"], cfg["N"], cfg["L"]
    if splitting == "lie" or dxd == 0:
        return _collide_all(_transport(F, n, cfg), F, cfg, tab, evaluator, integrator)
    h = cfg.get("dx", 1.0)
    d1 = transport.shift_delta_half(2 * n, N, L, cfg["dt"], h)
    d2 = transport.shift_delta_half(2 * n + 1, N, L, cfg["dt"], h)
    mid = _collide_all(_transport(F, n, cfg, delta=d1), F, cfg, tab, evaluator, integrator)
    return _transport(mid, n, cfg, delta=d2)


def homogeneous_step(f, tab, dt, tau=1.0, project=True, evaluator="fft", integrator="euler"):
    """0D (space-homogeneous) step of a batch [cells, (N,)*d]."""
    coll = collision.collide_fft if evaluator == "fft" else collision.collide_direct
    cfg = dict(dv=tab.d, N=tab.N, L=tab.L, dt=dt, tau=tau, project=project)
    out = np.empty_like(f)
    for c in range(f.shape[0]):
        out[c] = _collision_update(f[c], cfg, tab, coll, integrator)
    return out
