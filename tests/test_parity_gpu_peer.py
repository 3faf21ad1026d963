"""a2 fused into the step over peer memory (parallel.PeerHalo, include/fks.h fks_ipc_*): the step
kernel's transport gather reads the neighbour ranks' boundary planes in place.  Partitioned runs
must equal the single-domain run BITWISE.

* one process: every rank's context points fks_set_halo at the other ranks' buffers (device
  pointers on the same GPU), the ranks step in turn on one stream;
* two processes on the one GPU: the buffers are mapped with CUDA IPC handles exchanged over gloo,
  steps separated by host barriers (no kernel waits on another process's kernel).
"""
import os
import socket

import numpy as np
import pytest

import workloads
from oracle import transport

pytestmark = pytest.mark.gpu
P, G_, O = transport.PERIODIC, transport.GHOST, transport.OUTFLOW


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    if not _t.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return _t


def _problem(dxd, dv, M, N, bc, seed):
    L, h = 6.0, 0.1
    dt = 0.93 * h / (L - L / N)
    rng = np.random.default_rng(70 + seed)
    base = workloads.family("smooth", dv, N, L, 1, seed=seed)[0]
    F = (base[None] * rng.uniform(0.5, 1.5, int(np.prod(M)))[(...,) + (None,) * dv]).reshape(int(np.prod(M)), -1)
    ghosts = {f: workloads.family("smooth", dv, N, L, 1, seed=seed + 10 + f)[0].reshape(-1) for f in range(2 * dxd)
              if bc[f] == transport.GHOST}
    return L, h, dt, F, ghosts


def _ctx(fks, torch, dv, dxd, M, N, L, h, bc, ghosts, solid):
    c = fks.Context(dv, dxd, list(M), N, L, 8 if dv == 2 else 24, h=h, bc=bc)
    for face, g in ghosts.items():
        c.set_ghost(face, torch.from_numpy(g).cuda())
    if solid is not None:
        c.set_solid(solid)
    c.set_params(tau=0.5)
    return c


CASES = [
    (1, 3, [7], 8, [G_, O], 3, 3),
    (2, 3, [4, 6], 8, [O, O, P, P], 2, 9),       # periodic ring of 2
    (3, 3, [3, 2, 6], 8, [O, O, P, P, G_, O], 3, None),
    (2, 2, [5, 8], 16, [P, P, P, P], 4, 11),     # ring of 4
    (1, 3, [4], 64, [G_, O], 2, 1),              # 64^3
    (2, 3, [3, 5], 4, [G_, O, P, P], 2, 4),      # N = 4
]


@pytest.mark.parametrize("dxd,dv,M,N,bc,world,solid_at", CASES)
def test_peer_halo_one_process_bitwise(torch, dxd, dv, M, N, bc, world, solid_at):
    from paper_1608_08009_b200 import fks, parallel
    L, h, dt, F, ghosts = _problem(dxd, dv, M, N, bc, seed=dxd + world)
    solid = None
    if solid_at is not None:
        solid = np.zeros(tuple(M[::-1]), dtype=bool)
        solid.reshape(-1)[solid_at] = True
    ref = _ctx(fks, torch, dv, dxd, M, N, L, h, bc, ghosts, solid)
    slabs = [parallel.decompose(dxd, M, bc, world, r) for r in range(world)]
    G = torch.from_numpy(F).cuda()
    ctxs, bufs = [], []
    for s in slabs:
        sl = parallel.local_slice(s, solid.reshape(-1)) if solid is not None else None
        ctxs.append(_ctx(fks, torch, dv, dxd, s.M_local, N, L, h, s.local_bc(bc), ghosts,
                         None if sl is None else np.asarray(sl).reshape(tuple(s.M_local[::-1]))))
        loc = parallel.local_slice(s, G).contiguous()
        bufs.append([loc, torch.empty_like(loc)])
    n = F.shape[1]
    addrs = []
    for s in slabs:
        lq, hq = s.lower(), s.upper()
        addrs.append(parallel.peer_plane_addresses(
            s, n, [b.data_ptr() for b in bufs[lq]] if lq is not None else None,
            bufs[lq][0].shape[0] if lq is not None else 0,
            [b.data_ptr() for b in bufs[hq]] if hq is not None else None))
    p = 0
    for step in range(3):
        out = torch.empty_like(G)
        ref.step(G, out, dt)
        for r, (s, c) in enumerate(zip(slabs, ctxs)):
            lo, hi = addrs[r]
            c.set_halo_ptr(lo[p], hi[p])
            c.step(bufs[r][p], bufs[r][1 - p], dt)
        for r, s in enumerate(slabs):
            assert torch.equal(bufs[r][1 - p], parallel.local_slice(s, out)), (step, r)
        G = out
        p ^= 1
    for c in ctxs + [ref]:
        c.check()


def _ipc_worker(rank, world, port, case, result_path):
    import torch
    import torch.distributed as dist
    from paper_1608_08009_b200 import fks, parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    torch.cuda.set_device(0)
    dxd, dv, M, N, bc, _, solid_at = case
    L, h, dt, F, ghosts = _problem(dxd, dv, M, N, bc, seed=dxd + world)
    solid = None
    if solid_at is not None:
        solid = np.zeros(tuple(M[::-1]), dtype=bool)
        solid.reshape(-1)[solid_at] = True
    s = parallel.decompose(dxd, M, bc, world, rank)
    sl = parallel.local_slice(s, solid.reshape(-1)) if solid is not None else None
    ctx = _ctx(fks, torch, dv, dxd, s.M_local, N, L, h, s.local_bc(bc), ghosts,
               None if sl is None else np.asarray(sl).reshape(tuple(s.M_local[::-1])))
    loc = torch.from_numpy(np.ascontiguousarray(parallel.local_slice(s, F))).cuda()
    bufs = [loc, torch.empty_like(loc)]

    def host_barrier():
        torch.cuda.synchronize()
        dist.barrier()
    ph = parallel.PeerHalo(ctx, s, bufs, barrier=host_barrier)
    for _ in range(3):
        out = ph.step(dt)
    host_barrier()
    ctx.check()
    mine = out.cpu().numpy()
    every = [None] * world
    dist.all_gather_object(every, (s.lo, s.hi, mine))
    dist.barrier()  # every rank done reading its peers before anyone unmaps or frees
    ph.close()
    if rank == 0:
        ref = _ctx(fks, torch, dv, dxd, M, N, L, h, bc, ghosts, solid)
        a = torch.from_numpy(F).cuda()
        b = torch.empty_like(a)
        for _ in range(3):
            ref.step(a, b, dt)
            a, b = b, a
        want = a.cpu().numpy().reshape(tuple(M[::-1]) + (-1,))
        ok = all(np.array_equal(got.reshape((hi - lo,) + tuple(M[:-1][::-1]) + (-1,)), want[lo:hi])
                 for lo, hi, got in every)
        with open(result_path, "w") as fh:
            fh.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [CASES[0], CASES[2], CASES[4]])
def test_peer_halo_ipc_two_processes_bitwise(torch, case, tmp_path):
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    world = 2
    case = case[:5] + (world,) + case[6:]
    result = str(tmp_path / "result.txt")
    mp.start_processes(_ipc_worker, args=(world, port, case, result), nprocs=world, start_method="spawn")
    assert open(result).read() == "ok"
