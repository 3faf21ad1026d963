"""a2 inside libfks (fks_set_comm's exchange) on one GPU through the loopback communicator: the ranks'
contexts are driven in turn (every rank posts its planes, then every rank steps), and the slab-
partitioned run must equal the single-domain run BITWISE every step (partitioned
runs are compared bitwise) -- for C3/C4-shaped grids at full size and smaller 3D grids, with solids,
ghosts and periodic rings, for fks_step (interior || exchange, then boundary planes), fks_transport,
fks_step_bgk and the Heun scheme.  The NCCL path differs only in how the packed bytes move.
"""
import numpy as np
import pytest

import workloads
from oracle import transport

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    if not _t.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return _t


@pytest.fixture(scope="module")
def fks():
    from paper_1608_08009_b200 import fks as _f
    return _f


def _setup(torch, fks, dxd, dv, M, N, L, bc, world, A, h, ghosts, solid, tau=0.5, scheme=None, specular=False):
    from paper_1608_08009_b200 import parallel
    ref = fks.Context(dv, dxd, M, N, L, A, h=h, bc=bc)
    slabs = [parallel.decompose(dxd, M, bc, world, r) for r in range(world)]
    loop = fks.Loopback(world)
    ctxs = []
    for s in slabs:
        c = fks.Context(dv, dxd, list(s.M_local), N, L, A, h=h, bc=s.local_bc(bc))
        ctxs.append(c)
    for c in [ref] + ctxs:
        for face, g in ghosts.items():
            c.set_ghost(face, torch.from_numpy(g).cuda())
        c.set_params(tau=tau)
        if scheme is not None:
            c.set_scheme(*scheme)
        if specular:
            c.set_specular(True)
    if solid is not None:
        ref.set_solid(solid)
    for r, (s, c) in enumerate(zip(slabs, ctxs)):
        c.set_comm_loopback(loop, r)
        if solid is not None:
            c.set_solid(parallel.local_slice(s, solid.reshape(-1)))
    return ref, slabs, ctxs, loop


def _run(torch, fks, ref, slabs, ctxs, G, dt, steps, call):
    from paper_1608_08009_b200 import parallel
    n = G.shape[1]
    for c in ctxs:
        c.set_state(ref.get_state()[0], dt)   # dt fixed before the first post
    for step in range(steps):
        out = torch.empty_like(G)
        call(ref, G, out)
        locs = [parallel.local_slice(s, G).contiguous() for s in slabs]
        for c, loc in zip(ctxs, locs):
            c.halo_post(loc)
        for s, c, loc in zip(slabs, ctxs, locs):
            o = torch.empty_like(loc)
            call(c, loc, o)
            assert torch.equal(o, parallel.local_slice(s, out)), (step, s.rank)
        G = out
    return G


def _state(dxd, dv, M, N, L, bc, seed):
    rng = np.random.default_rng(40 + seed)
    base = workloads.family("smooth", dv, N, L, 1, seed=seed)[0]
    F = base[None] * rng.uniform(0.5, 1.5, int(np.prod(M)))[(...,) + (None,) * dv]
    ghosts = {f: workloads.family("smooth", dv, N, L, 1, seed=seed + 10 + f)[0] for f in range(2 * dxd)
              if bc[f] == transport.GHOST}
    return F.reshape(int(np.prod(M)), -1), ghosts


P, G_, O = transport.PERIODIC, transport.GHOST, transport.OUTFLOW


@pytest.mark.parametrize("dxd,dv,M,N,bc,world,solid_at", [
    (1, 3, [11], 8, [G_, G_], 3, None),
    (1, 2, [10], 16, [P, P], 2, 4),                      # periodic ring of 2: both neighbours the same peer
    (2, 3, [4, 7], 8, [G_, O, O, O], 2, 9),
    (2, 2, [5, 6], 16, [P, P, P, P], 3, None),
    (3, 3, [3, 2, 5], 8, [O, O, P, P, G_, O], 2, 7),
    (3, 3, [3, 3, 8], 8, [G_, O, O, O, P, P], 4, 20),    # ring of 4 along z
    (1, 3, [5], 64, [G_, O], 2, 2),                       # 64^3 (k_step3d64)
    (2, 3, [4, 6], 4, [G_, O, P, P], 3, 5),               # N = 4 (k_step_small), periodic ring of 3
    (2, 2, [5, 4], 4, [O, O, G_, O], 2, 7),
])
def test_loopback_step_bitwise(torch, fks, dxd, dv, M, N, bc, world, solid_at):
    L = 6.0
    h = 0.1
    dt = 0.93 * h / (L - L / N)
    F, ghosts = _state(dxd, dv, M, N, L, bc, seed=dxd + dv + world)
    solid = None
    if solid_at is not None:
        solid = np.zeros(tuple(M[::-1]), dtype=bool)
        solid.reshape(-1)[solid_at] = True
    A = 8 if dv == 2 else 24
    ref, slabs, ctxs, loop = _setup(torch, fks, dxd, dv, M, N, L, bc, world, A, h, ghosts, solid)
    G = torch.from_numpy(F).cuda()
    _run(torch, fks, ref, slabs, ctxs, G, dt, 3, lambda c, a, b: c.step(a, b, dt))
    # the exchange carried only the crossing slices
    n = N ** dv
    from paper_1608_08009_b200 import parallel
    for s, c in zip(slabs, ctxs):
        sent, inner, edge = c.comm_stats()
        assert 0 < sent < 2 * s.plane_cells * n * 8
        nsolid = 0 if solid is None else int(parallel.local_slice(s, solid.reshape(-1)).sum())
        assert inner + edge == int(np.prod(s.M_local)) - nsolid


@pytest.mark.parametrize("what", ["transport", "bgk", "heun"])
def test_loopback_other_calls_bitwise(torch, fks, what):
    dxd, dv, M, N, bc, world = 2, 3, [4, 6], 8, [G_, O, P, P], 3
    L, h = 6.0, 0.1
    dt = 0.93 * h / (L - L / N)
    F, ghosts = _state(dxd, dv, M, N, L, bc, seed=3)
    scheme = (fks.SPLIT_LIE, fks.TIME_HEUN) if what == "heun" else None
    ref, slabs, ctxs, loop = _setup(torch, fks, dxd, dv, M, N, L, bc, world, 24, h, ghosts, None, scheme=scheme)
    call = {"transport": lambda c, a, b: c.transport(a, b, dt),
            "bgk": lambda c, a, b: c.step_bgk(a, b, dt, fks.NU_RHO, 0.0),
            "heun": lambda c, a, b: c.step(a, b, dt)}[what]
    _run(torch, fks, ref, slabs, ctxs, torch.from_numpy(F).cuda(), dt, 3, call)


@pytest.mark.parametrize("name,world", [("C3", 4), ("C4", 4)])
def test_loopback_full_size_bitwise(torch, fks, name, world):
    """BASELINE C3 (400 cells, 4 slabs of 100) and C4 (100^2 cells with the solid boxes, 4 slabs of
    25 rows) at full size: two fused steps, partitioned == single domain bitwise."""
    c = workloads.config(name)
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    M = list(c["cells"][::-1])
    n = N ** dv
    nc = int(np.prod(M))
    v = workloads.initial_state(c, ncells=1).reshape(-1)[:n]
    s = 1.0 + 0.1 * np.random.default_rng(2).random(nc)
    G = torch.from_numpy(v[None, :].copy()).cuda() * torch.from_numpy(s[:, None].copy()).cuda()
    ref, slabs, ctxs, loop = _setup(torch, fks, dxd, dv, M, N, L, c["bc"], world, A, c["dx"],
                                    workloads.ghost_vectors(c), workloads.solid_mask(c), tau=c["tau"])
    _run(torch, fks, ref, slabs, ctxs, G, c["dt"], 2, lambda cc, a, b: cc.step(a, b, c["dt"]))


def test_comm_argument_errors(torch, fks):
    """fks_set_comm_loopback rejects a taken rank, a second comm and a rank out of range
    (include/fks.h); a step whose neighbour has not posted is FKS_E_STATE."""
    N, L, h = 8, 6.0, 0.1
    loop = fks.Loopback(2)
    a = fks.Context(3, 1, [4], N, L, 24, h=h, bc=[fks.BC_GHOST, fks.BC_HALO])
    b = fks.Context(3, 1, [4], N, L, 24, h=h, bc=[fks.BC_HALO, fks.BC_OUTFLOW])
    a.set_ghost(0, torch.zeros(N ** 3, dtype=torch.float64, device="cuda"))
    a.set_comm_loopback(loop, 0)
    with pytest.raises(fks.FksError) as ei:
        b.set_comm_loopback(loop, 0)
    assert ei.value.status == -1
    b.set_comm_loopback(loop, 1)
    with pytest.raises(fks.FksError):
        a.set_comm_loopback(loop, 1)
    dt = 0.9 * h / (L - L / N)
    f = torch.rand(4, N ** 3, dtype=torch.float64, device="cuda")
    a.set_state(0, dt)
    b.set_state(0, dt)
    a.halo_post(f)
    with pytest.raises(fks.FksError) as ei:
        a.step(f, torch.empty_like(f), dt)      # b has not posted step 0
    assert ei.value.status == -7
    c = fks.Context(3, 1, [4], N, L, 24, h=h, bc=[fks.BC_OUTFLOW, fks.BC_OUTFLOW])
    with pytest.raises(fks.FksError) as ei:
        c.set_comm_loopback(loop, 3)                # rank out of range
    assert ei.value.status == -1


@pytest.mark.parametrize("dxd,dv,M,N,bc,world,solid_cells", [
    # solids on both sides of every slab face (the walls straddle the partition)
    (2, 3, [5, 8], 8, [G_, O, O, O], 2, [(2, 3), (2, 4), (3, 4), (1, 0), (4, 7)]),
    (2, 2, [6, 9], 16, [P, P, P, P], 3, [(2, 2), (3, 3), (2, 5), (4, 6), (0, 8), (5, 0)]),
    (3, 3, [4, 3, 6], 8, [O, O, P, P, P, P], 3, [(1, 1, 1), (1, 1, 2), (2, 2, 3), (0, 0, 5), (3, 2, 0)]),
    (2, 3, [5, 6], 4, [G_, O, P, P], 2, [(2, 2), (2, 3), (1, 5), (3, 0)]),
])
def test_loopback_specular_bitwise(torch, fks, dxd, dv, M, N, bc, world, solid_cells):
    """NEXT-1 on a partitioned grid: specular walls that straddle slab faces reflect exactly as in
    one domain (the boundary planes' solid flags travel with the exchange), transport and fused
    steps bitwise equal to the single-domain run."""
    L, h = 6.0, 0.1
    dt = 0.93 * h / (L - L / N)
    F, ghosts = _state(dxd, dv, M, N, L, bc, seed=5 + dxd)
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    for cc in solid_cells:
        solid[tuple(reversed(cc))] = True
    A = 8 if dv == 2 else 24
    for call in ("transport", "step"):
        ref, slabs, ctxs, loop = _setup(torch, fks, dxd, dv, M, N, L, bc, world, A, h, ghosts, solid, specular=True)
        fn = {"transport": lambda c, a, b: c.transport(a, b, dt), "step": lambda c, a, b: c.step(a, b, dt)}[call]
        _run(torch, fks, ref, slabs, ctxs, torch.from_numpy(F).cuda(), dt, 3, fn)


def test_loopback_specular_C4_full_size(torch, fks):
    """The C4 geometry at full size with specular walls, 4 slabs of 25 rows: the boxes (rows 42-57)
    straddle the face between ranks 1 and 2; two fused steps, partitioned == single domain."""
    c = workloads.config("C4")
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    M = list(c["cells"][::-1])
    n = N ** dv
    nc = int(np.prod(M))
    v = workloads.initial_state(c, ncells=1).reshape(-1)[:n]
    s = 1.0 + 0.1 * np.random.default_rng(6).random(nc)
    G = torch.from_numpy(v[None, :].copy()).cuda() * torch.from_numpy(s[:, None].copy()).cuda()
    ref, slabs, ctxs, loop = _setup(torch, fks, dxd, dv, M, N, L, c["bc"], 4, A, c["dx"],
                                    workloads.ghost_vectors(c), workloads.solid_mask(c), tau=c["tau"], specular=True)
    _run(torch, fks, ref, slabs, ctxs, G, c["dt"], 2, lambda cc, a, b: cc.step(a, b, c["dt"]))


@pytest.mark.parametrize("dxd,dv,M,N,specular", [(1, 3, [6], 8, False), (2, 2, [4, 5], 16, False),
                                                 (3, 3, [3, 2, 4], 8, True), (2, 3, [3, 4], 4, True),
                                                 (1, 3, [3], 64, False)])
def test_nccl_single_rank_ring_bitwise(torch, fks, dxd, dv, M, N, specular):
    """The real NCCL path on one GPU: a one-rank communicator (fks_comm_unique_id + fks_set_comm,
    nranks = 1) whose slab axis is a periodic ring of one -- both HALO neighbours are the rank
    itself, so grouped ncclSend/ncclRecv to self carry the crossing slices (and, with specular walls,
    the solid flags) -- must reproduce the periodic single-domain run bitwise, three steps."""
    L, h = 6.0, 0.1
    dt = 0.93 * h / (L - L / N)
    bc = [P] * (2 * dxd)
    F, ghosts = _state(dxd, dv, M, N, L, bc, seed=50 + dxd)
    A = 8 if dv == 2 else 24
    ref = fks.Context(dv, dxd, M, N, L, A, h=h, bc=bc)
    bc_ring = list(bc)
    bc_ring[2 * (dxd - 1)] = bc_ring[2 * (dxd - 1) + 1] = fks.BC_HALO
    ring = fks.Context(dv, dxd, M, N, L, A, h=h, bc=bc_ring)
    if specular:
        solid = np.zeros(tuple(M[::-1]), dtype=bool)
        solid.reshape(-1)[[0, 5, len(solid.reshape(-1)) - 1]] = True   # on both slab-face planes
        for c in (ref, ring):
            c.set_solid(solid)
            c.set_specular(True)
    try:
        uid = fks.comm_unique_id()
    except fks.FksError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    ring.set_comm(uid, 0, 1)
    a = torch.from_numpy(F).cuda()
    ra, rb = a.clone(), torch.empty_like(a)
    b = torch.empty_like(a)
    for _ in range(3):
        ref.step(ra, rb, dt)
        ring.step(a, b, dt)
        ring.check()
        assert torch.equal(b, rb)
        ra, rb = rb, ra
        a, b = b, a
    sent, inner, edge = ring.comm_stats()
    assert sent > 0 and edge > 0
