"""FKS free transport as an exact integer shift per discrete velocity (oracle; tests only).

P:243-257 (eq. f_bar): the piecewise-constant function of velocity v_k is advected exactly,
f_bar_k^{*,n+1}(x) = f_bar_k^n(x - v_k dt); its discontinuities sit at x_{j+1/2} + n v_k dt
(they are "remembered" off the grid).  Sampling at the cell centre x_j
 therefore reads the piece whose origin cell is j + s^n_k with
s^n_k = floor(1/2 - n v_k dt / dx) (the particle reinterpretation P:547-573 tracks
only this one shift per velocity).  Storing the sampled values F^n_j = m[j + s^n] (an
Eulerian array) the transport from step n to n+1 is the gather

    f*_j[k] = F^n[j + delta_k][k],   delta_k = s^{n+1}_k - s^n_k  in {-1, 0, 1} at CFL <= 1.

Reading #16: both sides compute c = (v * dt) / dx, t = n * c, floor(0.5 - t) in fp64, no FMA.
Boundaries (reading #19): per face PERIODIC (wrap), GHOST (a fixed ghost vector, Dirichlet or
inflow), OUTFLOW (clamp to the boundary cell).  When several axes leave the domain the
lowest axis with a GHOST face wins; otherwise each axis is wrapped/clamped independently.
Shift per spatial axis a uses velocity component a (x_i += v_i dt).
Layout: F has shape spatial_shape + (N,)*dv; spatial_shape = (M_{dx-1}, .., M_0) (axis 0 fastest).
"""
import numpy as np

from . import grid

PERIODIC, GHOST, OUTFLOW = 0, 1, 2


def shift_s(n, N, L, dt, dx):
    """s^n_k = floor(0.5 - n * ((v_k * dt) / dx)) for the N nodes of one velocity axis."""
    v = grid.nodes_1d(N, L)
    c = (v * dt) / dx
    t = np.float64(n) * c
    return np.floor(0.5 - t).astype(np.int64)


def shift_delta(n, N, L, dt, dx):
    """delta_k = s^{n+1}_k - s^n_k."""
    return shift_s(n + 1, N, L, dt, dx) - shift_s(n, N, L, dt, dx)


def shift_s_half(p, N, L, dt, dx):
    """NEXT-4 (Strang splitting): the shift at the half-step position p (time p dt / 2),
    s = floor(0.5 - (p * c) * 0.5), c = (v_k dt) / dx.  For even p = 2n this is bitwise shift_s(n)
    (scaling by 2 and by 1/2 is exact in binary floating point)."""
    v = grid.nodes_1d(N, L)
    c = (v * dt) / dx
    t = (np.float64(p) * c) * 0.5
    return np.floor(0.5 - t).astype(np.int64)


def shift_delta_half(p, N, L, dt, dx):
    """delta_k from half-step position p to p + 1 (a transport over dt / 2)."""
    return shift_s_half(p + 1, N, L, dt, dx) - shift_s_half(p, N, L, dt, dx)


def gather(F, n, dxdim, dv, N, L, dt, dx, bc, ghosts=None, cells=None, delta=None):
    """f* from F^n.  bc: list of 2*dxdim face kinds [lo0, hi0, lo1, hi1, ...].
    ghosts: dict face -> ghost vector of shape (N,)*dv.  cells: optional flat cell indices; then
    only those cells are computed and returned as [len(cells), (N,)*dv].  delta: the per-node
    shift table to use instead of shift_delta(n) (Strang half steps)."""
    if dxdim == 0:
        return F.copy() if cells is None else F.reshape((-1,) + F.shape[dxdim:])[list(cells)].copy()
    sp_shape = F.shape[:dxdim]          # (M_{dx-1}, ..., M_0)
    M = sp_shape[::-1]                  # M[a] = cells along space axis a
    if delta is None:
        delta = shift_delta(n, N, L, dt, dx)
    vshape = (N,) * dv
    out = np.empty_like(F) if cells is None else None
    # velocity-axis index array per component a: component a is array axis dv-1-a
    kcomp = np.meshgrid(*([np.arange(N)] * dv), indexing="ij")
    kcomp = [kcomp[dv - 1 - a] for a in range(dv)]
    todo = range(int(np.prod(sp_shape))) if cells is None else list(cells)
    sub = None if cells is None else np.empty((len(todo),) + vshape)
    for pos, jflat in enumerate(todo):
        jidx = np.unravel_index(jflat, sp_shape)
        j = [jidx[dxdim - 1 - a] for a in range(dxdim)]
        src = []
        ghost_face = np.full(vshape, -1, dtype=np.int64)
        for a in range(dxdim):
            s = j[a] + delta[kcomp[a]]
            lo_out, hi_out = s < 0, s >= M[a]
            for face, mask in ((2 * a, lo_out), (2 * a + 1, hi_out)):
                kind = bc[face]
                if kind == PERIODIC:
                    s = np.where(mask, s % M[a], s)
                elif kind == OUTFLOW:
                    s = np.where(mask, np.clip(s, 0, M[a] - 1), s)
                elif kind == GHOST:
                    ghost_face = np.where(mask & (ghost_face < 0), face, ghost_face)
                    s = np.where(mask, np.clip(s, 0, M[a] - 1), s)
                else:
                    raise ValueError(kind)
            src.append(s)
        idx = tuple(src[dxdim - 1 - b] for b in range(dxdim)) + tuple(
            np.broadcast_to(g, vshape) for g in np.meshgrid(*([np.arange(N)] * dv), indexing="ij"))
        vals = F[idx]
        if ghosts is not None:
            for face, gv in ghosts.items():
                vals = np.where(ghost_face == face, gv, vals)
        if sub is None:
            out[jidx] = vals
        else:
            sub[pos] = vals
    return out if sub is None else sub


def gather_specular(F, n, dxd, dv, N, L, dt, dx, bc, ghosts, solid, cells=None, delta=None):
    """NEXT-1: f* with specular reflection at solid cells ("reflective boundary conditions",
    S:430-438 apply_solid_reflection; reading #23 of DESIGN.md).

    Forward picture: a particle of velocity index k moves axis by axis (axis 0 first) by its
    shift; when the next cell along an axis is solid it is reflected instead (v_a -> -v_a, on the
    symmetric lattice k_a -> N-1-k_a) and stays.  The gather inverts that map, so in a closed box
    it is a permutation of the fluid values (mass and energy conserved exactly).  For a fluid cell
    j and arrived velocity k, undo the axes in reverse order (dxd-1 .. 0) from c = j:
      the candidate origin along a is c + delta_a(k_a) e_a (wrapped on a PERIODIC face); if it is an
      in-domain solid cell the particle was reflected there: k_a -> N-1-k_a and c stays;
      otherwise c moves to it.
    The value is then read as in gather() from the source j + (the shifts of the axes that were not
    reflected), with the face rules (GHOST / OUTFLOW / PERIODIC), at the mirrored index k'.  Without
    solids this is exactly gather().  Solid cells keep their values.  Plain scalar loops.
    cells: optional flat cell indices; then only those cells are computed and returned as
    [len(cells), (N,)*dv] (F may then be any object with .shape and integer-tuple indexing)."""
    sp_shape = F.shape[:dxd]
    M = sp_shape[::-1]
    if delta is None:
        delta = shift_delta(n, N, L, dt, dx)
    out = np.empty_like(F) if cells is None else np.empty((len(cells),) + (N,) * dv)

    def in_domain_solid(cell):                               # cell: list of dxd coordinates
        if any(c < 0 or c >= M[a] for a, c in enumerate(cell)):
            return False
        return bool(solid[tuple(cell[dxd - 1 - b] for b in range(dxd))])

    todo = range(int(np.prod(sp_shape))) if cells is None else list(cells)
    for pos, jflat in enumerate(todo):
        jidx = np.unravel_index(jflat, sp_shape)
        oidx = jidx if cells is None else (pos,)
        if solid[jidx]:
            out[oidx] = F[jidx]
            continue
        j = [jidx[dxd - 1 - a] for a in range(dxd)]
        for kidx in np.ndindex(*((N,) * dv)):
            kc = [kidx[dv - 1 - a] for a in range(dv)]      # velocity component a
            d = [int(delta[kc[a]]) for a in range(dxd)]
            flip = [False] * dv
            c = list(j)
            for a in reversed(range(dxd)):
                if d[a] == 0:
                    continue
                nb = list(c)
                nb[a] = c[a] + d[a]
                if bc[2 * a if d[a] < 0 else 2 * a + 1] == PERIODIC:
                    nb[a] %= M[a]
                if in_domain_solid(nb):
                    flip[a], d[a] = True, 0
                else:
                    c = nb
            # the source after the face rules (as gather(): lowest axis with a ghost face wins)
            s, gface = list(j), -1
            for a in range(dxd):
                v = j[a] + d[a]
                if v < 0 or v >= M[a]:
                    face = 2 * a if v < 0 else 2 * a + 1
                    kind = bc[face]
                    if kind == PERIODIC:
                        v %= M[a]
                    else:
                        if kind == GHOST and gface < 0:
                            gface = face
                        v = min(max(v, 0), M[a] - 1)
                s[a] = v
            kp = [N - 1 - kc[a] if flip[a] else kc[a] for a in range(dv)]
            kpidx = tuple(kp[dv - 1 - b] for b in range(dv))
            if gface >= 0:
                val = ghosts[gface][kpidx]
            else:
                val = F[tuple(s[dxd - 1 - b] for b in range(dxd)) + kpidx]
            out[oidx + kidx] = val
    return out
