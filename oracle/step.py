"""One first-order split step (oracle; test infrastructure only).

P:226-233: Lie splitting, transport first then collision.
P:259-275 (eq. f_coll): forward Euler on the cell-centred values, f^{n+1} = f* + dt Q(f*).
P:909: the rescaled equation d_t f + v.grad f = Q(f)/tau.
P:319-320 + reading #13: the collision output is projected to zero moments.
Solid cells (reading #19) keep their values; the collision is skipped there.
"""
import numpy as np

from . import collision, projection, transport


def step(F, n, cfg, tab, evaluator="fft"):
    """F^{n+1} from F^n.  cfg: dict with dx_dim, dv, N, L, dt, dx, tau, bc, ghosts, solid, project."""
    dxd, dv, N, L = cfg["dx_dim"], cfg["dv"], cfg["N"], cfg["L"]
    fstar = transport.gather(F, n, dxd, dv, N, L, cfg["dt"], cfg.get("dx", 1.0), cfg.get("bc"),
                             cfg.get("ghosts"))
    coll = collision.collide_fft if evaluator == "fft" else collision.collide_direct
    sp_shape = F.shape[:dxd]
    solid = cfg.get("solid")
    out = np.empty_like(F)
    for jflat in range(int(np.prod(sp_shape)) if dxd else 1):
        jidx = np.unravel_index(jflat, sp_shape) if dxd else ()
        if solid is not None and solid[jidx]:
            out[jidx] = F[jidx]
            continue
        fj = fstar[jidx]
        Q = coll(fj, tab)
        if cfg.get("project", True):
            Q = projection.project_zero_moments(Q, dv, N, L)
        out[jidx] = fj + (cfg["dt"] / cfg["tau"]) * Q
    return out


def homogeneous_step(f, tab, dt, tau=1.0, project=True, evaluator="fft"):
    """0D (space-homogeneous) step of a batch [cells, (N,)*d]."""
    coll = collision.collide_fft if evaluator == "fft" else collision.collide_direct
    out = np.empty_like(f)
    for c in range(f.shape[0]):
        Q = coll(f[c], tab)
        if project:
            Q = projection.project_zero_moments(Q, tab.d, tab.N, tab.L)
        out[c] = f[c] + (dt / tau) * Q
    return out
