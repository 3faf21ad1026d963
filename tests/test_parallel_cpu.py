"""Multi-rank host logic on CPU (gloo, world size 2-3): slab decomposition, face kinds, and the
halo exchange, checked end to end against the oracle's single-domain transport gather."""
import datetime
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import transport
from paper_1608_08009_b200 import parallel
from paper_1608_08009_b200.fks import BC_GHOST, BC_HALO, BC_OUTFLOW, BC_PERIODIC


def test_decompose_covers_planes():
    for m in [7, 12, 48, 100]:
        for world in [1, 2, 3, 4, 8]:
            if world > m:
                continue
            slabs = [parallel.decompose(2, (5, m), [0, 0, 2, 2], world, r) for r in range(world)]
            assert slabs[0].lo == 0 and slabs[-1].hi == m
            assert all(a.hi == b.lo for a, b in zip(slabs, slabs[1:]))
            sizes = [s.hi - s.lo for s in slabs]
            assert max(sizes) - min(sizes) <= 1


def test_local_face_kinds():
    s = [parallel.decompose(3, (4, 4, 9), [BC_GHOST, BC_OUTFLOW] * 3, 3, r) for r in range(3)]
    assert s[0].local_bc([BC_GHOST, BC_OUTFLOW] * 3)[4:] == [BC_GHOST, BC_HALO]
    assert s[1].local_bc([BC_GHOST, BC_OUTFLOW] * 3)[4:] == [BC_HALO, BC_HALO]
    assert s[2].local_bc([BC_GHOST, BC_OUTFLOW] * 3)[4:] == [BC_HALO, BC_OUTFLOW]
    ring = [parallel.decompose(1, (10,), [BC_PERIODIC, BC_PERIODIC], 2, r) for r in range(2)]
    assert ring[0].lower() == 1 and ring[1].upper() == 0
    assert ring[0].local_bc([BC_PERIODIC, BC_PERIODIC]) == [BC_HALO, BC_HALO, 0, 0, 0, 0]
    single = parallel.decompose(1, (10,), [BC_PERIODIC, BC_PERIODIC], 1, 0)
    assert single.local_bc([BC_PERIODIC, BC_PERIODIC])[:2] == [BC_PERIODIC, BC_PERIODIC]


CASES = {
    # dx, dv, M (axis 0 fastest), N, L, global bc
    "2d_space_3d_vel": (2, 3, (4, 7), 8, 5.0, [BC_GHOST, BC_OUTFLOW, BC_OUTFLOW, BC_OUTFLOW]),
    "1d_ring": (1, 2, (9,), 8, 4.0, [BC_PERIODIC, BC_PERIODIC]),
    "3d_space": (3, 3, (3, 2, 6), 8, 5.0, [BC_OUTFLOW, BC_OUTFLOW, BC_PERIODIC, BC_PERIODIC, BC_GHOST, BC_OUTFLOW]),
}


def _global_state(case):
    dx, dv, M, N, L, bc = CASES[case]
    rng = np.random.default_rng(3)
    F = rng.random(tuple(M[::-1]) + (N,) * dv)
    ghosts = {f: rng.random((N,) * dv) for f in range(2 * dx) if bc[f] == BC_GHOST}
    return F, ghosts


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        dx, dv, M, N, L, bc = CASES[case]
        n = N ** dv
        F, ghosts = _global_state(case)
        Fg = torch.from_numpy(F.reshape(-1, n))
        slab = parallel.decompose(dx, M, bc, world, rank)
        local = parallel.local_slice(slab, Fg).clone()
        hx = parallel.HaloExchange(slab, n, "cpu")
        lo, hi = hx.exchange(local)
        elo, ehi = parallel.halos_from_global(slab, Fg)
        ok = True
        for got, exp in ((lo, elo), (hi, ehi)):
            ok &= (got is None) == (exp is None)
            if got is not None:
                ok &= bool(torch.equal(got, exp))
        # FKS transport of the slab with the exchanged halo planes equals the global transport
        h, dt = 0.1, 0.09 / (L - L / N)
        pieces = ([lo] if lo is not None else []) + [local] + ([hi] if hi is not None else [])
        ext = torch.cat(pieces).numpy()
        Mext = list(M)
        Mext[dx - 1] = ext.shape[0] // slab.plane_cells
        ext = ext.reshape(tuple(Mext[::-1]) + (N,) * dv)
        bc_ext = list(bc)
        if slab.world > 1 and slab.periodic:
            bc_ext[2 * (dx - 1)] = bc_ext[2 * (dx - 1) + 1] = BC_OUTFLOW  # the halos carry the wrap
        for step in range(3):
            ref = transport.gather(F, step, dx, dv, N, L, dt, h, bc, ghosts).reshape(-1, n)
            got = transport.gather(ext, step, dx, dv, N, L, dt, h, bc_ext, ghosts).reshape(-1, n)
            off = slab.plane_cells if lo is not None else 0
            mine = got[off:off + local.shape[0]]
            ok &= bool(np.array_equal(mine, ref[slab.lo * slab.plane_cells:slab.hi * slab.plane_cells]))
        out[rank] = ok
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case,world", [("2d_space_3d_vel", 2), ("1d_ring", 2), ("3d_space", 3)])
def test_halo_exchange_gloo(case, world):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world, start_method="spawn")
    assert dict(out) == {r: True for r in range(world)}


def _worker_libplan(rank, world, port, case, out):
    """a2 as libfks does it (fks_set_comm): per step only the velocity slices the library's plan
    names (fks_host_halo_slices) are sent, packed [plane cells][slices][other components]; the
    neighbour planes start as NaN, so a slice the transport needs but the plan omits would show."""
    from paper_1608_08009_b200 import fks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        dx, dv, M, N, L, bc = CASES[case]
        n = N ** dv
        F, ghosts = _global_state(case)
        slab = parallel.decompose(dx, M, bc, world, rank)
        pc = slab.plane_cells
        vshape = (N,) * dv
        ax = dv - 1 - (dx - 1)           # array axis of velocity component dx - 1 (layout [kz, ky, kx])
        local = parallel.local_slice(slab, F.reshape(-1, *vshape))
        h, dt = 0.1, 0.09 / (L - L / N)
        ok = True
        for step in range(4):
            down, up = fks.host_halo_slices(step, N, L, dt, h)
            d = transport.shift_delta(step, N, L, dt, h)
            ok &= set(down) == set(np.nonzero(d > 0)[0]) and set(up) == set(np.nonzero(d < 0)[0])
            first, last = local[:pc], local[-pc:]
            send_lo = np.ascontiguousarray(np.take(first, down, axis=1 + ax))
            send_hi = np.ascontiguousarray(np.take(last, up, axis=1 + ax))
            lo_r, hi_r = slab.lower(), slab.upper()
            rlo = np.empty(send_hi.shape) if lo_r is not None else None   # lower's last plane, `up` slices
            rhi = np.empty(send_lo.shape) if hi_r is not None else None   # upper's first plane, `down` slices
            ops = []
            if hi_r is not None:
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(send_hi), hi_r, None, 0))
            if lo_r is not None:
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(send_lo), lo_r, None, 1))
            if lo_r is not None:
                t_lo = torch.from_numpy(rlo)
                ops.append(dist.P2POp(dist.irecv, t_lo, lo_r, None, 0))
            if hi_r is not None:
                t_hi = torch.from_numpy(rhi)
                ops.append(dist.P2POp(dist.irecv, t_hi, hi_r, None, 1))
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            pieces = []
            if lo_r is not None:
                plane = np.full((pc,) + vshape, np.nan)
                idx = [slice(None)] * (1 + dv)
                idx[1 + ax] = up
                plane[tuple(idx)] = t_lo.numpy()
                pieces.append(plane)
            pieces.append(local)
            if hi_r is not None:
                plane = np.full((pc,) + vshape, np.nan)
                idx = [slice(None)] * (1 + dv)
                idx[1 + ax] = down
                plane[tuple(idx)] = t_hi.numpy()
                pieces.append(plane)
            ext = np.concatenate(pieces)
            Mext = list(M)
            Mext[dx - 1] = ext.shape[0] // pc
            ext = ext.reshape(tuple(Mext[::-1]) + vshape)
            bc_ext = list(bc)
            if slab.world > 1 and slab.periodic:
                bc_ext[2 * (dx - 1)] = bc_ext[2 * (dx - 1) + 1] = BC_OUTFLOW
            ref = transport.gather(F, step, dx, dv, N, L, dt, h, bc, ghosts).reshape(-1, n)
            got = transport.gather(ext, step, dx, dv, N, L, dt, h, bc_ext, ghosts).reshape(-1, n)
            off = pc if lo_r is not None else 0
            mine = got[off:off + local.shape[0]]
            ok &= bool(np.array_equal(mine, ref[slab.lo * pc:slab.hi * pc]))
            # bytes on the wire per step = what fks_get_comm_stats reports: pc x slices x N^(dv-1) x 8
            ok &= send_lo.nbytes == pc * len(down) * N ** (dv - 1) * 8
        out[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("2d_space_3d_vel", 2), ("1d_ring", 2), ("3d_space", 3)])
def test_libfks_halo_plan_gloo(case, world):
    """The library's exchange plan (only delta != 0 slices cross a face) is sufficient: the oracle's
    transport on the slab plus the partially filled neighbour planes equals the global transport
    bitwise, over several steps, for 2-3 ranks on CPU (gloo)."""
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker_libplan, args=(world, _free_port(), case, out), nprocs=world, start_method="spawn")
    assert dict(out) == {r: True for r in range(world)}


@pytest.mark.parametrize("world,periodic", [(3, False), (4, True), (1, True)])
def test_peer_plane_addresses(world, periodic):
    """PeerHalo's pointer arithmetic against the global layout: with the ranks' buffers laid out
    back to back as one global array, the lower neighbour's last plane and the upper neighbour's
    first plane are exactly the global planes next to the slab (halos_from_global)."""
    M, n = [3, 2, 11], 5
    bc = [BC_OUTFLOW] * 4 + ([BC_PERIODIC] * 2 if periodic else [BC_GHOST, BC_OUTFLOW])
    slabs = [parallel.decompose(3, M, bc, world, r) for r in range(world)]
    pc = slabs[0].plane_cells
    # buffer b of rank r lives at base 10**6 * (2 r + b + 1) bytes; its planes are the slab's planes
    base = {(r, b): 10 ** 6 * (2 * r + b + 1) for r in range(world) for b in range(2)}
    for s in slabs:
        lo_q, hi_q = s.lower(), s.upper()
        lo, hi = parallel.peer_plane_addresses(
            s, n, [base[(lo_q, b)] for b in range(2)] if lo_q is not None else None,
            int(np.prod(slabs[lo_q].M_local)) if lo_q is not None else 0,
            [base[(hi_q, b)] for b in range(2)] if hi_q is not None else None)
        for b in range(2):
            if lo_q is None:
                assert lo[b] is None
            else:
                q = slabs[lo_q]
                # the global plane just below s.lo is plane (hi - 1) of rank lo_q
                assert s.lo - 1 == q.hi - 1 or (periodic and s.lo == 0 and q.hi == M[2])
                assert lo[b] == base[(lo_q, b)] + ((q.hi - q.lo) - 1) * pc * n * 8
            if hi_q is None:
                assert hi[b] is None
            else:
                assert hi[b] == base[(hi_q, b)]
