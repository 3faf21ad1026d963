"""Multi-GPU plumbing: slab decomposition of physical space and the halo exchange (a2).

The paper distributes "spatial degrees of freedom over computational nodes, keeping on every
node a complete set of velocity space points", slices along one axis, and exchanges ghost
cells after each step (Fig. mpi-decomp).  Here one process drives one GPU; the slab
axis is the slowest space axis (axis dx-1); each rank owns a contiguous range of planes with
all N^dv velocities; per step each rank sends its first / last plane to its lower / upper
neighbour (torch.distributed P2P: NCCL over NVLink on GPUs, gloo on CPU for the tests) and
the step kernel reads sources outside the slab from those planes (FKS_BC_HALO faces).  The
FKS shift is at most one cell per step at CFL <= 1 (reading #15), so one plane suffices.

0D ensembles (C1/C2) need none of this: ranks own disjoint cell batches and never communicate
on the data path (bench.py, weak scaling).

Nothing here computes any part of the method: it partitions indices and moves bytes.
"""
from dataclasses import dataclass

from .fks import BC_HALO, BC_PERIODIC


@dataclass
class Slab:
    dx: int
    M_global: tuple      # cells per space axis, axis 0 fastest
    rank: int
    world: int
    lo: int              # first global plane index owned along the slab axis
    hi: int              # one past the last
    periodic: bool = False  # the slab axis is periodic in the global problem (ring of ranks)

    @property
    def axis(self):
        return self.dx - 1

    @property
    def M_local(self):
        m = list(self.M_global)
        m[self.axis] = self.hi - self.lo
        return tuple(m)

    @property
    def plane_cells(self):
        p = 1
        for a in range(self.dx - 1):
            p *= self.M_global[a]
        return p

    def lower(self):
        """Rank owning the plane below lo (None at a non-periodic domain face)."""
        return self._neighbour(-1)

    def upper(self):
        return self._neighbour(+1)

    def _neighbour(self, d):
        r = self.rank + d
        if 0 <= r < self.world:
            return r
        return (r % self.world) if self.periodic else None

    def local_bc(self, bc_global):
        """Face kinds of the local grid: slab-axis faces shared with another rank become HALO."""
        bc = list(bc_global) + [0] * (6 - len(bc_global))
        lo_face, hi_face = 2 * self.axis, 2 * self.axis + 1
        if self.world > 1:
            if self.lower() is not None:
                bc[lo_face] = BC_HALO
            if self.upper() is not None:
                bc[hi_face] = BC_HALO
        return bc


def decompose(dx, M_global, bc_global, world, rank):
    """Near-equal contiguous slabs along the slowest axis (first ranks get the extra plane)."""
    if dx < 1:
        raise ValueError("slab decomposition needs dx >= 1")
    m = M_global[dx - 1]
    if world > m:
        raise ValueError("more ranks than planes")
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    periodic = bc_global[2 * (dx - 1)] == BC_PERIODIC and bc_global[2 * (dx - 1) + 1] == BC_PERIODIC
    return Slab(dx=dx, M_global=tuple(M_global), rank=rank, world=world, lo=lo, hi=hi, periodic=periodic)


def local_slice(slab, f_global):
    """The rank's part of a global [cells..., n] array laid out [planes][plane cells][n]."""
    pc = slab.plane_cells
    return f_global[slab.lo * pc:slab.hi * pc]


def halos_from_global(slab, f_global):
    """(lo, hi) neighbour planes taken from a global array (single-process emulation/tests)."""
    pc = slab.plane_cells
    m = slab.M_global[slab.axis]
    lo = hi = None
    if slab.lower() is not None:
        p = (slab.lo - 1) % m
        lo = f_global[p * pc:(p + 1) * pc]
    if slab.upper() is not None:
        p = slab.hi % m
        hi = f_global[p * pc:(p + 1) * pc]
    return lo, hi


class HaloExchange:
    """Per-step exchange of boundary planes with torch.distributed batched P2P."""

    def __init__(self, slab, n, device, dtype=None, group=None):
        import torch
        self.slab, self.group = slab, group
        dtype = dtype or torch.float64
        pc = slab.plane_cells
        self.lo = torch.empty(pc, n, device=device, dtype=dtype) if slab.lower() is not None else None
        self.hi = torch.empty(pc, n, device=device, dtype=dtype) if slab.upper() is not None else None
        self.pc, self.n = pc, n

    def exchange(self, f_local):
        """Fill self.lo / self.hi from the neighbours; f_local is [local cells, n] (contiguous)."""
        import torch.distributed as dist
        pc = self.pc
        f_local = f_local.reshape(-1, self.n)
        first, last = f_local[:pc], f_local[-pc:]
        # Fixed order per peer pair (NCCL matches P2P in issue order; gloo also uses the tags):
        # data moving up (my last plane -> upper's lo halo) before data moving down.
        ops = []
        lo_r, hi_r = self.slab.lower(), self.slab.upper()
        if hi_r is not None:
            ops.append(dist.P2POp(dist.isend, last.contiguous(), hi_r, self.group, 0))
        if lo_r is not None:
            ops.append(dist.P2POp(dist.isend, first.contiguous(), lo_r, self.group, 1))
        if lo_r is not None:
            ops.append(dist.P2POp(dist.irecv, self.lo, lo_r, self.group, 0))
        if hi_r is not None:
            ops.append(dist.P2POp(dist.irecv, self.hi, hi_r, self.group, 1))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return self.lo, self.hi


def init_libfks_comm(ctx, rank, world, group=None, device=None):
    """a2 inside libfks (fks_set_comm): rank 0 draws the NCCL unique id, torch.distributed broadcasts
    the 128 bytes, every rank builds the library's own communicator.  Afterwards ctx.step does the
    exchange itself (only the crossing velocity slices, overlapped with the interior cells)."""
    import torch
    import torch.distributed as dist
    from . import fks
    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(fks.comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0, group=group)
    ctx.set_comm(bytes(t.cpu().numpy().tobytes()), rank, world)


class DistributedStep:
    """fks_step on one rank's slab with a torch.distributed halo exchange of whole planes in front
    (a2 -> a1..a9).  The production path is init_libfks_comm (the exchange inside the library);
    this class remains for CPU (gloo) checks of the host logic."""

    def __init__(self, ctx, slab, n, device, group=None):
        self.ctx, self.x = ctx, HaloExchange(slab, n, device, group=group)

    def __call__(self, f_in, f_out, dt):
        import torch
        # the exchange runs on torch's current stream: put the step on the same stream so the
        # kernel reads the halo planes after the receive landed and the next exchange cannot
        # overwrite them while the kernel still runs
        if f_in.is_cuda:
            self.ctx.set_stream(torch.cuda.current_stream(f_in.device))
        lo, hi = self.x.exchange(f_in)
        self.ctx.set_halo(lo, hi)
        self.ctx.step(f_in, f_out, dt)


def peer_plane_addresses(slab, n, lower_bases, lower_cells, upper_bases, itemsize=8):
    """Byte addresses of the neighbour planes a rank's HALO faces read, per buffer parity:
    lo[b] = the lower neighbour's LAST plane of its buffer b (its local cells `lower_cells`),
    hi[b] = the upper neighbour's FIRST plane.  None where the slab face is a domain face."""
    plane = slab.plane_cells * n * itemsize
    lo = [None, None] if lower_bases is None else [b + lower_cells * n * itemsize - plane for b in lower_bases]
    hi = [None, None] if upper_bases is None else list(upper_bases)
    return lo, hi


class PeerHalo:
    """a2 fused into the step over peer memory (include/fks.h fks_ipc_*).

    Every rank keeps its state in two ping-pong buffers; once, the ranks exchange CUDA IPC handles
    of them (torch.distributed.all_gather_object) and map their neighbours' buffers.  Each step
    then points fks_set_halo at the neighbours' boundary planes of the current parity, so the step
    kernel's transport gather reads the sources across a slab face straight from the peer GPU
    (NVLink / NVSwitch): no pack, send, receive or unpack kernels, no staging copy.  Ordering is
    one barrier per step (`barrier`, default a 1-element all_reduce on the current stream, which
    NCCL orders with the kernels): step n + 1 reads the neighbours' step-n output, and their step
    n + 2 overwrites that buffer only after everyone passed the next barrier.  Specular walls across
    a face need the neighbours' solid flags: use init_libfks_comm for those runs."""

    def __init__(self, ctx, slab, bufs, group=None, barrier=None):
        import torch
        import torch.distributed as dist
        from . import fks
        self.ctx, self.slab, self.bufs = ctx, slab, bufs
        n = bufs[0][0].numel()
        ncells = bufs[0].shape[0]
        mine = ([fks.ipc_handle(b) for b in bufs], ncells)
        every = [None] * slab.world
        dist.all_gather_object(every, mine, group=group)
        self._mapped = {}

        def bases(q):
            if q is None:
                return None
            if q == slab.rank:  # a periodic ring of one rank: its own buffers
                return [b.data_ptr() for b in bufs]
            if q not in self._mapped:
                self._mapped[q] = [fks.ipc_open(h) for h, _ in every[q][0]]
            return [base + off for base, (_, off) in zip(self._mapped[q], every[q][0])]

        lo_q, hi_q = slab.lower(), slab.upper()
        self.lo, self.hi = peer_plane_addresses(slab, n, bases(lo_q), every[lo_q][1] if lo_q is not None else 0,
                                                bases(hi_q))
        if barrier is None:
            token = torch.zeros(1, device=bufs[0].device)

            def barrier():
                dist.all_reduce(token, group=group)
        self.barrier = barrier
        self.parity = 0
        ctx.set_stream(torch.cuda.current_stream(bufs[0].device))

    def step(self, dt):
        """One fused step: bufs[parity] -> bufs[1 - parity]; returns the output buffer."""
        self.barrier()
        b = self.parity
        self.ctx.set_halo_ptr(self.lo[b], self.hi[b])
        self.ctx.step(self.bufs[b], self.bufs[1 - b], dt)
        self.parity ^= 1
        return self.bufs[1 - b]

    def close(self):
        from . import fks
        for bases in self._mapped.values():
            for b in bases:
                fks.ipc_close(b)
        self._mapped = {}
