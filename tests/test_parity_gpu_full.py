"""GPU parity at the BASELINE configs' full sizes and at the edges the round-1 review listed:
C5 (48^3 cells, > 2^31 state elements) sampled cell by cell, a 10-step C2 run with the error
growth reported, the C4 geometry at N = 32 with specular walls, fks_step_host on a spatial grid,
the CFL guard on partitioned grids, thin periodic axes at CFL > 1 and the specular source
resolution next to OUTFLOW faces.  Same criteria as tests/test_parity_gpu.py (§8(c.5)):
per cell max_k |f_gpu - f_orc| / max_k |f_orc| <= 1e-11; transport bitwise.
"""
import numpy as np
import pytest

import workloads
from oracle import collision, projection, step as ostep, tables, transport

pytestmark = pytest.mark.gpu
TOL = 1e-11


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


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def _flat(c, xyz):
    """Flat local cell index of space coordinates (x, y, z) (axis 0 fastest)."""
    M = c["cells"][::-1]
    j, stride = 0, 1
    for a, v in enumerate(xyz):
        j += v * stride
        stride *= M[a]
    return j


def _scaled_state(torch, c, seed):
    """F[j] = s_j * m (m the config's uniform Maxwellian, s_j = 1 + 0.1 U[0,1)) built on the device
    by one broadcast multiply (bitwise the numpy product), plus the lazy host twin for the oracle."""
    m = workloads.initial_state(c, ncells=1).reshape((-1,) + (c["N"],) * c["dv"])[0]
    s = 1.0 + 0.1 * np.random.default_rng(seed).random(tuple(c["cells"]))
    Fd = dev(torch, m.reshape(1, -1)) * dev(torch, s.reshape(-1, 1))
    return Fd, workloads.ScaledField(m, s)


def _check_sampled(got_rows, sample, fstar, solid_flat, Fh, c, tab):
    N, dv = c["N"], c["dv"]
    sp = tuple(c["cells"])
    for i, cell in enumerate(sample):
        if solid_flat is not None and solid_flat[cell]:
            np.testing.assert_array_equal(got_rows[i], Fh[np.unravel_index(cell, sp)])
            continue
        Q = projection.project_zero_moments(collision.collide_fft(fstar[i], tab), dv, N, c["L"])
        ref = fstar[i] + (c["dt"] / c["tau"]) * Q
        err = np.max(np.abs(got_rows[i] - ref)) / np.max(np.abs(ref))
        assert err <= TOL, (c["name"], cell, err)


def test_full_size_C5_sampled(torch, fks):
    """BASELINE configs[4] (3Dx3D, 48^3 cells, 12^3 solid cuboid, inflow at x = 0, outflow
    elsewhere; 3.6e9 state elements, so offsets above 2^31 are exercised) at full size in bench.py's
    launch configuration: one fused step, cells on every face kind, next to the cuboid, inside it
    and past flat index 2^31 / n = 65536, each against the oracle."""
    c = workloads.config("C5")
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    M = list(c["cells"][::-1])
    Fd, Fh = _scaled_state(torch, c, seed=5)
    ghosts = workloads.ghost_vectors(c)
    solid = workloads.solid_mask(c)
    ctx = fks.Context(dv, dxd, M, N, L, A, h=c["dx"], bc=c["bc"])
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    ctx.set_params(tau=c["tau"])
    out = torch.empty_like(Fd)
    ctx.step(Fd, out, c["dt"])
    ctx.check()
    pts = [(0, 0, 0), (47, 0, 0), (0, 47, 47), (47, 47, 47), (17, 20, 20), (30, 24, 24), (20, 17, 25),
           (24, 24, 30), (29, 29, 17), (20, 20, 20), (5, 40, 40), (0, 24, 47), (31, 30, 29)]
    sample = [_flat(c, p) for p in pts]
    assert max(sample) * N ** 3 > 2 ** 31 and solid.reshape(-1)[_flat(c, (20, 20, 20))]
    got = host(out[sample])
    del out, Fd
    torch.cuda.empty_cache()
    fstar = transport.gather(Fh, 0, dxd, dv, N, L, c["dt"], c["dx"], c["bc"], ghosts, cells=sample)
    _check_sampled(got.reshape((-1,) + (N,) * dv), sample, fstar, solid.reshape(-1), Fh, c,
                   tables.build_tables(dv, N, L))


def test_C2_ten_steps_growth(torch, fks, capsys):
    """§8(c.5): C2 cells (Test 1.3 two-Gaussian relaxation, 32^3, 24-design) stepped 10 times on
    the GPU and by the oracle; every step within 1e-11, the per-step worst error reported."""
    c = workloads.config("C2")
    N, L = c["N"], c["L"]
    nc = 6
    f = workloads.initial_state(c, ncells=nc, start=1000)
    ctx = fks.Context(3, 0, [nc], N, L, 24)
    a, b = dev(torch, f), torch.empty(nc, N, N, N, dtype=torch.float64, device="cuda")
    tab = tables.build_tables(3, N, L)
    ref = f.copy()
    growth = []
    for s in range(10):
        ctx.step(a, b, c["dt"])
        a, b = b, a
        ref = ostep.homogeneous_step(ref, tab, c["dt"])
        got = host(a)
        growth.append(max(np.max(np.abs(got[i] - ref[i])) / np.max(np.abs(ref[i])) for i in range(nc)))
    with capsys.disabled():
        print("\nC2 10-step parity growth: " + " ".join(f"{e:.2e}" for e in growth))
    assert max(growth) <= TOL


def test_C4_geometry_specular_n32(torch, fks):
    """NEXT-1 at full size: the C4 geometry (Test 3.2 boxes, 100^2 cells, N = 32^3) with specular
    reflection at the solid cells: one fused step, fluid cells touching the boxes (faces
    and corners) and far from them against the oracle's gather_specular + collision."""
    c = workloads.config("C4")
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    M = list(c["cells"][::-1])
    Fd, Fh = _scaled_state(torch, c, seed=4)
    ghosts = workloads.ghost_vectors(c)
    solid = workloads.solid_mask(c)
    ctx = fks.Context(dv, dxd, M, N, L, A, h=c["dx"], bc=c["bc"])
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    ctx.set_solid(solid)
    ctx.set_specular(True)
    ctx.set_params(tau=c["tau"])
    out = torch.empty_like(Fd)
    ctx.step(Fd, out, c["dt"])
    ctx.check()
    # fluid cells with a solid 8-neighbour (walls and box corners), plus a few others
    ys, xs = np.nonzero(solid)
    cand = set()
    for y, x in zip(ys, xs):
        for dy in (-1, 0, 1):
            for dx_ in (-1, 0, 1):
                yy, xx = y + dy, x + dx_
                if 0 <= yy < M[1] and 0 <= xx < M[0] and not solid[yy, xx]:
                    cand.add(yy * M[0] + xx)
    cand = sorted(cand)
    rng = np.random.default_rng(44)
    sample = [int(v) for v in rng.choice(cand, size=6, replace=False)] + [0, 99, 9999, int(ys[0] * M[0] + xs[0])]
    got = host(out[sample]).reshape((-1,) + (N,) * dv)
    fstar = transport.gather_specular(Fh, 0, dxd, dv, N, L, c["dt"], c["dx"], c["bc"], ghosts, solid, cells=sample)
    _check_sampled(got, sample, fstar, solid.reshape(-1), Fh, c, tables.build_tables(dv, N, L))


@pytest.mark.parametrize("dxd,dv,M,N,bc,solid_cell", [
    (1, 3, [40], 8, [transport.GHOST, transport.GHOST], None),
    (2, 2, [9, 7], 16, [transport.GHOST, transport.OUTFLOW, transport.OUTFLOW, transport.OUTFLOW], 20),
    (1, 3, [6], 64, [transport.GHOST, transport.OUTFLOW], 3),
    (0, 3, [9], 64, [], None),                           # homogeneous: the pipelined host path
])
def test_step_host_spatial(torch, fks, dxd, dv, M, N, bc, solid_cell):
    """fks_step_host (host buffers, one H2D + step + D2H) on spatial grids equals fks_step bitwise."""
    L = 6.0
    rng = np.random.default_rng(3)
    shape = tuple(M[::-1]) + (N,) * dv
    F = workloads.family("smooth", dv, N, L, int(np.prod(M)), seed=9).reshape(shape)
    F = F * (1.0 + 0.1 * rng.random(tuple(M[::-1])))[(...,) + (None,) * dv]
    h = 0.1
    dt = 0.9 * h / (L - L / N)
    ghosts = {f: workloads.family("smooth", dv, N, L, 1, seed=30 + f)[0] for f in range(2 * dxd)
              if bc[f] == transport.GHOST}
    outs = []
    for use_host in (False, True):
        ctx = fks.Context(dv, dxd, M, N, L, 8 if dv == 2 else 24, h=h, bc=bc)
        for face, g in ghosts.items():
            ctx.set_ghost(face, dev(torch, g))
        if solid_cell is not None:
            sm = np.zeros(tuple(M[::-1]), dtype=bool)
            sm.reshape(-1)[solid_cell] = True
            ctx.set_solid(sm)
        if use_host:
            hin = torch.from_numpy(F.copy()).pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            ctx.step_host(hin, hout, dt)
            ctx.step_host(hout, hin, dt)
            outs.append(hin.numpy().copy())
        else:
            a, b = dev(torch, F), torch.empty(shape, dtype=torch.float64, device="cuda")
            ctx.step(a, b, dt)
            ctx.step(b, a, dt)
            outs.append(host(a))
    np.testing.assert_array_equal(outs[0], outs[1])


def test_cfl_guard_on_partitioned_grid(torch, fks):
    """A HALO face carries one plane (halo width 1, reading #15): a dt whose shift along the slab
    axis exceeds one cell is refused (FKS_E_UNSUPPORTED) by fks_step, fks_transport and
    fks_step_bgk, with nothing enqueued; the same dt is accepted without a HALO face."""
    N, L, h = 8, 5.0, 0.1
    dt = 1.7 * h / (L - L / N)
    assert np.max(np.abs(transport.shift_delta(0, N, L, dt, h))) >= 2
    f = dev(torch, workloads.family("smooth", 3, N, L, 12, seed=1)).reshape(12, -1)
    o = torch.empty_like(f)
    ctx = fks.Context(3, 2, [3, 4], N, L, 24, h=h, bc=[0, 0, fks.BC_HALO, fks.BC_OUTFLOW])
    ctx.set_halo(f[:3].contiguous(), None)
    for call in (lambda: ctx.step(f, o, dt), lambda: ctx.transport(f, o, dt), lambda: ctx.step_bgk(f, o, dt, 0, 0.0)):
        n0 = ctx.launch_count()
        with pytest.raises(fks.FksError) as ei:
            call()
        assert ei.value.status == -2 and ctx.launch_count() == n0
    assert ctx.get_state()[0] == 0
    ok = fks.Context(3, 2, [3, 4], N, L, 24, h=h, bc=[0, 0, fks.BC_OUTFLOW, fks.BC_OUTFLOW])
    ok.transport(f, o, dt)
    ok.check()
    # CFL <= 1 on the partitioned grid is fine
    dt1 = 0.9 * h / (L - L / N)
    ctx2 = fks.Context(3, 2, [3, 4], N, L, 24, h=h, bc=[0, 0, fks.BC_HALO, fks.BC_OUTFLOW])
    ctx2.set_halo(f[:3].contiguous(), None)
    ctx2.transport(f, o, dt1)
    ctx2.check()


@pytest.mark.parametrize("M,cfl", [([1, 3], 1.8), ([2, 3], 2.6), ([3, 2], 2.6)])
def test_transport_thin_periodic_axis_high_cfl(torch, fks, M, cfl):
    """Periodic axes thinner than the shift (|delta| > M_a): the wrap is a true modulo, bitwise
    equal to the oracle's gather over several steps (general gather kernel, CFL > 1)."""
    dxd, dv, N, L = 2, 3, 8, 5.0
    bc = [transport.PERIODIC] * 4
    h = 0.1
    dt = cfl * h / (L - L / N)
    rng = np.random.default_rng(17)
    F = rng.random(tuple(M[::-1]) + (N,) * dv)
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(4):
        ctx.transport(a, b, dt)
        a, b = b, a
        ref = transport.gather(ref, s, dxd, dv, N, L, dt, h, bc, None)
    np.testing.assert_array_equal(host(a), ref)


@pytest.mark.parametrize("solid_xyz", [(1, 3, 0), (2, 0, 1), (0, 3, 2), (3, 3, 2), (1, 1, 1), (2, 3, 1)])
@pytest.mark.parametrize("cfl", [0.93, 1.8])
def test_specular_next_to_outflow_faces(torch, fks, solid_xyz, cfl):
    """Specular reflection on a 4x4x3 all-OUTFLOW box with one solid cell: a source resolution that
    leaves the domain along one axis never looks up (or aliases) a solid cell through another
    (every coordinate must be inside the domain); bitwise vs the oracle's gather_specular."""
    dxd, dv, N, L = 3, 3, 8, 5.0
    M = [4, 4, 3]
    bc = [transport.OUTFLOW] * 6
    h = 0.1
    dt = cfl * h / (L - L / N)
    rng = np.random.default_rng(23)
    F = rng.random(tuple(M[::-1]) + (N,) * dv)
    solid = np.zeros(tuple(M[::-1]), dtype=bool)
    x, y, z = solid_xyz
    solid[z, y, x] = True
    ctx = fks.Context(dv, dxd, M, N, L, 24, h=h, bc=bc)
    ctx.set_solid(solid)
    ctx.set_specular(True)
    a, b = dev(torch, F), torch.empty_like(dev(torch, F))
    ref = F.copy()
    for s in range(2):
        ctx.transport(a, b, dt)
        a, b = b, a
        ref = transport.gather_specular(ref, s, dxd, dv, N, L, dt, h, bc, {}, solid)
    np.testing.assert_array_equal(host(a), ref)


def test_configuration_and_state_errors(torch, fks):
    """The configuration calls and the steps report misuse with the documented status and enqueue
    nothing (include/fks.h): FKS_E_INVAL for bad arguments, FKS_E_STATE for out-of-order use."""
    import ctypes
    N, L, h = 8, 6.0, 0.1
    bc = [fks.BC_GHOST, fks.BC_OUTFLOW]
    ctx = fks.Context(3, 1, [5], N, L, 24, h=h, bc=bc)
    f = torch.rand(5, N ** 3, dtype=torch.float64, device="cuda")
    o = torch.empty_like(f)
    lib, hnd = ctx._lib, ctx.handle
    dt = 0.9 * h / (L - L / N)
    n0 = ctx.launch_count()
    for call, status in (
        (lambda: lib.fks_set_params(hnd, 0.0, 0.0, 0.0, 1), -1),
        (lambda: lib.fks_set_params(hnd, -1.0, 0.0, 0.0, 1), -1),
        (lambda: lib.fks_set_ghost(hnd, 6, ctypes.c_void_p(f.data_ptr())), -1),
        (lambda: lib.fks_set_ghost(hnd, 0, None), -1),
        (lambda: lib.fks_set_dirs(hnd, None, None, 0), -1),
        (lambda: lib.fks_set_state(hnd, -1, dt), -1),
        (lambda: lib.fks_moments(hnd, ctypes.c_void_p(f.data_ptr()), None, None, None), -1),
        (lambda: lib.fks_step(hnd, None, ctypes.c_void_p(o.data_ptr()), ctypes.c_double(dt)), -1),
        (lambda: lib.fks_transport(hnd, ctypes.c_void_p(f.data_ptr()), None, ctypes.c_double(dt)), -1),
        # in place is allowed; here it still fails on the unset ghost face, launching nothing
        (lambda: lib.fks_step(hnd, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(f.data_ptr()), ctypes.c_double(dt)), -7),
        (lambda: lib.fks_step(hnd, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(o.data_ptr()), ctypes.c_double(0.0)), -1),
        (lambda: lib.fks_step(hnd, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(o.data_ptr()), ctypes.c_double(dt)), -7),  # ghost face 0 never set
    ):
        assert call() == status, status
    with pytest.raises(fks.FksError):
        ctx.set_params(tau=0.0)           # the binding raises on the same status
    assert ctx.launch_count() == n0
    ctx.set_ghost(0, f[0].contiguous())
    ctx.step(f, o, dt)
    with pytest.raises(fks.FksError) as ei:
        ctx.step(o, f, 1.5 * dt)          # dt is fixed per run (reading #15)
    assert ei.value.status == -7
    n, dt_ = ctx.get_state()
    assert n == 1 and dt_ == dt
    ctx.set_state(7, dt)                  # resume: the shifts are pure functions of n
    ctx.step(o, f, dt)
    assert ctx.get_state()[0] == 8
    ctx.check()


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_full_size_256_cells(torch, fks, name):
    """§8(c.5) evaluator rule: at least 256 sampled cells per 3D config against the oracle's cpu_fft
    (C3: all 400 cells), one fused step at full size in bench.py's launch configuration."""
    c = workloads.config(name)
    N, L, A, dv, dxd = c["N"], c["L"], c["A"], c["dv"], c["dx_dim"]
    tab = tables.build_tables(dv, N, L)
    rng = np.random.default_rng(256)
    if dxd == 0:
        nc = c["cells"][0]
        f = workloads.initial_state(c)
        ctx = fks.Context(dv, 0, [nc], N, L, A)
        fin = dev(torch, f)
        out = torch.empty_like(fin)
        ctx.step(fin, out, c["dt"])
        ctx.check()
        sample = sorted(rng.choice(nc, size=256, replace=False).tolist())
        got = host(out[sample])
        ref = ostep.homogeneous_step(f[sample], tab, c["dt"], c["tau"])
        for i in range(256):
            assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), sample[i]
        return
    M = list(c["cells"][::-1])
    nc = int(np.prod(M))
    Fd, Fh = _scaled_state(torch, c, seed=256)
    ghosts = workloads.ghost_vectors(c)
    solid = workloads.solid_mask(c)
    ctx = fks.Context(dv, dxd, M, N, L, A, h=c["dx"], bc=c["bc"])
    for face, g in ghosts.items():
        ctx.set_ghost(face, dev(torch, g))
    if solid is not None:
        ctx.set_solid(solid)
    ctx.set_params(tau=c["tau"])
    out = torch.empty_like(Fd)
    ctx.step(Fd, out, c["dt"])
    ctx.check()
    sample = list(range(nc)) if nc <= 400 else sorted(rng.choice(nc, size=256, replace=False).tolist())
    got = host(out[sample]).reshape((-1,) + (N,) * dv)
    del out, Fd
    torch.cuda.empty_cache()
    fstar = transport.gather(Fh, 0, dxd, dv, N, L, c["dt"], c["dx"], c["bc"], ghosts, cells=sample)
    _check_sampled(got, sample, fstar, None if solid is None else solid.reshape(-1), Fh, c, tab)
