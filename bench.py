"""Benchmark of the fused FKS + fast-spectral step on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

One "step" = one fks_step over the whole batch (all §8(a) rows the config has: transport with
boundaries for C3-C5, collision a4-a7, projection a8, Euler a9).  Default workload: BASELINE.json
configs[1] = C2 (0Dx3D hard-sphere two-Gaussian relaxation ensemble, Nv = 32^3, A = 24 spherical
7-design directions), 4096 cells per GPU (1 GiB state, larger than L2), weak scaling across
ranks with no collective on the data path.  Prints ONE JSON line on rank 0.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "collision evals/s (Nv=32³, M dirs) and phase-space updates/s at 1/2/4/8 B200"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = {3: os.path.join(ROOT, "profiles", "r01_ncu_k_step3d.json"),
               2: os.path.join(ROOT, "profiles", "r01_ncu_k_step2d.json")}


def hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from MEASURED_PEAKS.json, else the guide's fallback."""
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 7700.0


def dram_traffic(dv, ncells, config=None):
    """dram__bytes_read + dram__bytes_write per launch from the committed `ncu --set full` capture
    of the dominant kernel on this config (profiles/r02_ncu_<kernel>_<config>.json: per-cell figure x
    cells of this launch), else the round-1 capture, else None.  Returns (bytes, source)."""
    kern = "k_step3d" if dv == 3 else "k_step2d"
    paths = ([os.path.join(ROOT, "profiles", f"r02_ncu_{kern}_{config}.json")] if config else []) + [NCU_SUMMARY.get(dv)]
    for path in paths:
        if path and os.path.exists(path):
            with open(path) as fh:
                return json.load(fh)["dram_bytes_per_cell"] * ncells, os.path.relpath(path, ROOT)
    return None, None
# FP64 DFMA peak: the SUSTAINED measurement committed in profiles/r02_peaks.json (>= 8 s of DFMA
# back to back on this pool's B200, clocks logged; tools/microbench/mb_dsmem.cu), else the figure
# derived from unit counts and clocks (B200_PROFILING.md: 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz).
FP64_PEAK_DERIVED = 148 * 64 * 2 * 1.965e9 / 1e12
PEAKS_R02 = os.path.join(ROOT, "profiles", "r02_peaks.json")


def fp64_peak():
    """(TFLOP/s, source) of the FP64 roofline denominator."""
    try:
        with open(PEAKS_R02) as fh:
            d = json.load(fh)
        return float(d["fp64_tflops_sustained"]), d.get("fp64_source", os.path.relpath(PEAKS_R02, ROOT))
    except (OSError, KeyError, ValueError):
        return FP64_PEAK_DERIVED, "derived: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"


FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = fp64_peak()


def flops_per_cell(dv, N, A):
    """SURVEY §8(a) / App. A.9 algorithmic flops per cell-step: (A+1) 5 n log2 n + (9A + 25) n."""
    n = N ** dv
    return (A + 1) * 5 * n * math.log2(n) + (9 * A + 25) * n


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--cells", type=int, default=0, help="override cells per GPU (0D configs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-spatial-secondary", action="store_true", help="skip the C4 fused-step and 64^3 secondary figures")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self):
        self.rows, self.proc = [], None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", os.environ.get("LOCAL_RANK", "0")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def wait_first(self, timeout=3.0):
        """Block until the sampler delivered its first row (nvidia-smi start-up), so that the
        timed region that follows is covered; returns the row count (the region's first index)."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.01)
        self.mark = len(self.rows)
        return self.mark

    def stop(self):
        # a timed region shorter than the 100 ms sampling period may end before any sample lands in
        # it: take the next one (the clock right at the end of the region) rather than none
        t0 = time.time()
        while self.proc and len(self.rows) <= getattr(self, "mark", 0) and time.time() - t0 < 0.5:
            time.sleep(0.01)
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
        rows = self.rows[getattr(self, "mark", 0):] or self.rows  # the timed region's samples
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


# ------------------------------------------------------------------ oracle (CPU) timing
def _oracle_worker(args):
    os.environ["OMP_NUM_THREADS"] = "1"
    name, start, count, evaluator = args
    import workloads
    from oracle import step as ostep, tables
    c = workloads.config(name)
    if c["dx_dim"] == 0:
        f = workloads.initial_state(c, ncells=count, start=start)
    else:  # spatial configs: the per-cell collision step dominates; time it on smooth cells
        f = workloads.family("smooth", c["dv"], c["N"], c["L"], count, seed=start)
    tab = tables.build_tables(c["dv"], c["N"], c["L"], A=c["A"]) if c["dv"] == 2 else tables.build_tables(3, c["N"], c["L"])
    t0 = time.perf_counter()
    ostep.homogeneous_step(f, tab, c["dt"], c["tau"], evaluator=evaluator)
    return time.perf_counter() - t0


def direct_timing():
    """the oracle's literal O(n^2 (A+1)) bilinear form (the paper's "naive" evaluation,
    P:414) timed on one 2D 32^2 cell (A = 8) and one 3D 16^3 cell (A = 24), single core; the 3D 32^3
    figure is extrapolated by (32768 / 4096)^2 = 64 (the cost is n^2 (A+1) complex MACs)."""
    import numpy as np
    import workloads
    from oracle import collision, tables
    out = {}
    for dv, N, L, A in ((2, 32, 9.0, 8), (3, 16, 7.0, 24)):
        f = workloads.family("smooth", dv, N, L, 1, seed=1)[0]
        tab = tables.build_tables(dv, N, L, A=A) if dv == 2 else tables.build_tables(3, N, L)
        t0 = time.perf_counter()
        collision.collide_direct(f, tab)
        out[f"direct_{dv}d_{N}_s_per_cell"] = time.perf_counter() - t0
    out["direct_3d_32_s_per_cell_extrapolated"] = out["direct_3d_16_s_per_cell"] * 64
    return out


def oracle_rate(name, seconds=15.0, cores=None):
    """cells/s of the oracle's fast evaluator (collide_fft + projection + Euler, numpy) over a
    bounded sample, one single-threaded worker per host core."""
    import multiprocessing as mp
    import workloads
    c = workloads.config(name)
    cores = cores or os.cpu_count() or 1
    # calibrate: one cell on one core
    t1 = _oracle_worker((name, 0, 1, "fft"))
    per_worker = max(1, int(seconds / max(t1, 1e-6) / 2))
    tot = per_worker * cores
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        times = pool.map(_oracle_worker, [(name, (i * per_worker) % max(1, c["cells"][0] - per_worker), per_worker,
                                           "fft") for i in range(cores)])
    wall = max(times)  # workers run concurrently; each times only its own step loop
    return tot / wall, cores, tot, wall


def n64_secondary(L, A, tau, dt, stream, reps, ncells=128):
    """The 64^3 velocity grid (k_step3d64: a 64-CTA group per cell), not a BASELINE config: the
    fused step on 128 homogeneous cells of the default workload's velocity box, CUDA events."""
    import torch
    import workloads
    from paper_1608_08009_b200 import fks
    N = 64
    n = N ** 3
    f = workloads.family("smooth", 3, N, L, 8, seed=5)
    fa = torch.from_numpy(f).cuda().repeat(ncells // 8, 1, 1, 1).contiguous()
    fb = torch.empty_like(fa)
    ctx = fks.Context(3, 0, [ncells], N, L, A)
    ctx.set_params(tau=tau)
    ctx.set_stream(stream)
    ctx.step(fa, fb, dt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        ctx.step(fa, fb, dt)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ctx.check()
    ctx.close()
    del fa, fb
    torch.cuda.empty_cache()
    ach = flops_per_cell(3, N, A) * ncells / (ms * 1e-3) / 1e12
    return {"value": ncells / (ms * 1e-3), "unit": "cells/s", "ms": ms, "fp64_frac": ach / FP64_PEAK_TFLOPS,
            "phase_space_updates_per_s": ncells * n / (ms * 1e-3),
            "what": f"fks_step on {ncells} homogeneous cells of a 64^3 velocity grid (k_step3d64), A = {A}"}


def spatial_secondary(name, stream, reps):
    """The transport-fused path on a spatial config (default: C4, 2Dx3D 100^2 cells with the solid
    boxes, inflow/outflow): fks_step (a1..a9 fused, ghosts, solids) timed with CUDA events, plus
    fks_transport alone (HBM-bound)."""
    import numpy as np
    import torch
    import workloads
    from paper_1608_08009_b200 import fks
    c = workloads.config(name)
    dv, N, A = c["dv"], c["N"], c["A"]
    n = N ** dv
    M = list(c["cells"][::-1])
    nc = int(np.prod(M))
    ctx = fks.Context(dv, c["dx_dim"], M, N, c["L"], A, h=c["dx"], bc=c["bc"])
    for face, g in workloads.ghost_vectors(c).items():
        ctx.set_ghost(face, torch.from_numpy(g).cuda())
    solid = workloads.solid_mask(c)
    nfl = nc
    if solid is not None:
        ctx.set_solid(solid)
        nfl = nc - int(solid.sum())
    ctx.set_params(tau=c["tau"])
    ctx.set_stream(stream)
    v = torch.from_numpy(workloads.initial_state(c, ncells=1).reshape(-1)[:n].copy()).cuda()
    s = torch.from_numpy(1.0 + 0.1 * np.random.default_rng(1).random(nc)).cuda()
    fa = (v[None, :] * s[:, None]).contiguous()
    fb = torch.empty_like(fa)
    dt = c["dt"]

    def timed(fn, k):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k
    ms = timed(lambda: ctx.step(fa, fb, dt), reps)
    ms_t = timed(lambda: ctx.transport(fa, fb, dt), reps)
    ctx.check()
    ach = flops_per_cell(dv, N, A) * nfl / (ms * 1e-3) / 1e12
    gbs = 2 * nc * n * 8 / (ms_t * 1e-3) / 1e9
    ctx.close()
    del fa, fb
    torch.cuda.empty_cache()
    return {"value": nfl / (ms * 1e-3), "unit": "cells/s", "ms": ms, "fp64_frac": ach / FP64_PEAK_TFLOPS,
            "phase_space_updates_per_s": nfl * n / (ms * 1e-3),
            "transport_only": {"ms": ms_t, "hbm_gbs": gbs, "hbm_frac": gbs / hbm_peak()},
            "what": f"{name} fks_step fused with FKS transport (ghost inflow, outflow, {nc - nfl} solid cells), "
                    f"{nfl} fluid cells, {reps} steps; transport_only = fks_transport alone (16 B per update)"}


# ------------------------------------------------------------------ main
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import workloads
    c = workloads.config(a.config)
    dv, N, A = c["dv"], c["N"], c["A"]
    n = N ** dv

    if a.impl == "reference":
        if rank != 0:
            return
        steps, warm = a.steps, a.warmup
        budget = min(20.0, max(3.0, 120.0 / max(1, steps + warm)))
        for _ in range(warm):
            oracle_rate(a.config, seconds=min(budget, 5.0))
        rates, cores_used, sample = [], 0, 0
        for _ in range(steps):
            r, cores_used, tot, wall = oracle_rate(a.config, seconds=budget)
            rates.append(r)
            sample = tot
        val = sum(rates) / len(rates)
        ms = 1e3 * c["cells"][0] / val
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "cells/s", "n_gpus": a.gpus,
                "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{a.config} oracle step (collide_fft + projection + Euler, numpy fp64)",
                           "cells_per_gpu": c["cells"][0], "Nv": N, "dv": dv, "M_dirs": A},
                "phase_space_updates_per_s": val * n,
                "cpu_baseline": {"value": val, "unit": "cells/s", "cores": cores_used, "kind": "oracle",
                                 "sample": f"{sample} cells of {a.config} per step on {cores_used} single-threaded "
                                           f"workers (ms_per_step extrapolated to {c['cells'][0]} cells)"},
                "e2e": {"value": val, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import numpy as np
    import torch
    from paper_1608_08009_b200 import fks

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    dt = c["dt"]
    if c["dx_dim"] == 0:
        ncells = a.cells or c["cells"][0]
        # synthetic input: 256 distinct generated cells tiled to the batch (numpy generation of
        # 4096 cells takes longer than the timed run); every cell still runs the full path
        base = workloads.initial_state(c, ncells=min(ncells, 256), start=(rank * 256) % c["cells"][0])
        reps = (ncells + base.shape[0] - 1) // base.shape[0]
        F = np.concatenate([base] * reps)[:ncells]
        ctx = fks.Context(dv, 0, [ncells], N, c["L"], A)
        fa = torch.from_numpy(F).cuda()
        nfluid_local = ncells
        stepper = None
        scaling = "weak"
    else:
        from paper_1608_08009_b200 import parallel
        dxd = c["dx_dim"]
        Mg = tuple(c["cells"][::-1])  # axis 0 fastest
        bc = c["bc"]
        slab = parallel.decompose(dxd, Mg, bc, world, rank)
        ctx = fks.Context(dv, dxd, list(slab.M_local), N, c["L"], A, h=c["dx"], bc=slab.local_bc(bc))
        for face, g in workloads.ghost_vectors(c).items():
            ctx.set_ghost(face, torch.from_numpy(g).cuda())
        solid = workloads.solid_mask(c)
        sl = parallel.local_slice(slab, solid.reshape(-1)) if solid is not None else None
        if sl is not None:
            ctx.set_solid(sl)
        nfluid_local = int(sl.size - sl.sum()) if sl is not None else int(np.prod(slab.M_local))
        if c["name"] == "C3":
            F = parallel.local_slice(slab, workloads.initial_state(c).reshape(-1, n))
            fa = torch.from_numpy(np.ascontiguousarray(F)).cuda()
        else:  # uniform initial state: one generated vector broadcast on the device
            v = torch.from_numpy(workloads.initial_state(c, ncells=1).reshape(-1)[:n].copy()).cuda()
            fa = v.expand(int(np.prod(slab.M_local)), n).contiguous()
            F = None
        if world > 1:  # a2 inside libfks: NCCL communicator of the library, crossing slices only
            parallel.init_libfks_comm(ctx, rank, world)
        stepper = None
        scaling = "strong"
        ncells = int(np.prod(slab.M_local))
    ctx.set_params(tau=c["tau"])
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)
    fb = torch.empty_like(fa)

    def one_step(x, y):
        if stepper is not None:
            stepper(x, y, dt)
        else:
            ctx.step(x, y, dt)

    for _ in range(a.warmup):
        one_step(fa, fb)
        fa, fb = fb, fa
    ctx.check()
    clocks = Clocks()
    clocks.start()
    time.sleep(0.3)
    clocks.wait_first()
    launches0 = ctx.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(a.steps):
        evs[i][0].record(stream)
        one_step(fa, fb)
        evs[i][1].record(stream)
        fa, fb = fb, fa
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ctx.check()
    launches = ctx.launch_count() - launches0
    ms_total = t_start.elapsed_time(t_end)
    kern_ms = [s.elapsed_time(e) for s, e in evs]
    if dist:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / a.steps
    nfluid = nfluid_local
    if dist:
        t = torch.tensor([float(nfluid_local)], device="cuda")
        dist.all_reduce(t)
        nfluid = int(t.item())
    else:
        nfluid = nfluid_local
    value = nfluid * a.steps / (ms_total * 1e-3)  # fluid cells collided per second, all ranks
    fl = flops_per_cell(dv, N, A)
    kern_avg_ms = sum(kern_ms) / len(kern_ms)
    achieved = fl * nfluid_local / (kern_avg_ms * 1e-3) / 1e12

    # ---- secondary figures (not the headline): collide-only and transport-only rates ---------
    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    extra = {}
    if stepper is None:
        reps = max(1, min(a.steps, 5))
        ms_c = timed(lambda: ctx.collide(fa, fb), reps)
        extra["collide_only"] = {"value": nfluid_local / (ms_c * 1e-3), "unit": "cells/s", "ms": ms_c,
                                 "what": "fks_collide (a4-a7, Q only), same cells"}
        if dv == 3 and c["dx_dim"] == 0:  # the 8x8 product grid (A = 64) as secondary
            ctx64 = fks.Context(dv, 0, [ncells], N, c["L"], 64)
            ctx64.set_params(tau=c["tau"])
            ctx64.set_stream(stream)
            ms_64 = timed(lambda: ctx64.step(fa, fb, dt), reps)
            ctx64.check()
            ach64 = flops_per_cell(dv, N, 64) * ncells / (ms_64 * 1e-3) / 1e12
            extra["A64_step"] = {"value": ncells / (ms_64 * 1e-3), "unit": "cells/s", "ms": ms_64,
                                 "fp64_frac": ach64 / FP64_PEAK_TFLOPS,
                                 "what": "fks_step with the 8x8 product direction grid (A = 64), same cells"}
            ctx64.close()
        if c["dx_dim"] > 0:
            ms_t = timed(lambda: ctx.transport(fa, fb, dt), reps)
            gbs = 2 * ncells * n * 8 / (ms_t * 1e-3) / 1e9
            peak = hbm_peak()
            extra["transport_only"] = {"value": ncells / (ms_t * 1e-3), "unit": "cells/s", "ms": ms_t,
                                       "hbm_gbs": gbs, "hbm_peak_gbs": peak,
                                       "hbm_frac": gbs / peak if peak else None,
                                       "what": "fks_transport (a1+a3, 16 B per phase-space update), HBM-bound"}
        # NEXT-2: the BGK step on the same cells (nu = rho), HBM-bound (16 B per update)
        ctxb = fks.Context(dv, c["dx_dim"], [ncells] if c["dx_dim"] == 0 else list(slab.M_local), N, c["L"], A,
                           **({} if c["dx_dim"] == 0 else dict(h=c["dx"], bc=slab.local_bc(c["bc"]))))
        if c["dx_dim"] > 0:
            for face, g in workloads.ghost_vectors(c).items():
                ctxb.set_ghost(face, torch.from_numpy(g).cuda())
            if sl is not None:
                ctxb.set_solid(sl)
        ctxb.set_params(tau=c["tau"])
        ctxb.set_stream(stream)
        ms_b = timed(lambda: ctxb.step_bgk(fa, fb, dt, fks.NU_RHO, 0.0), reps)
        ctxb.check()
        gbs = 2 * nfluid_local * n * 8 / (ms_b * 1e-3) / 1e9
        extra["bgk_step"] = {"value": nfluid_local / (ms_b * 1e-3), "unit": "cells/s", "ms": ms_b, "hbm_gbs": gbs,
                             "hbm_frac": gbs / hbm_peak(),
                             "what": "NEXT-2 fks_step_bgk (transport + conservative Maxwellian + Euler, nu = rho)"}
        ctxb.close()
        rho = torch.empty(ncells, dtype=torch.float64, device=fa.device)
        uu = torch.empty(ncells, dv, dtype=torch.float64, device=fa.device)
        TT = torch.empty(ncells, dtype=torch.float64, device=fa.device)
        ms_m = timed(lambda: ctx.moments(fa, rho, uu, TT), reps)
        gbs = ncells * n * 8 / (ms_m * 1e-3) / 1e9
        extra["moments_only"] = {"value": ncells / (ms_m * 1e-3), "unit": "cells/s", "ms": ms_m, "hbm_gbs": gbs,
                                 "hbm_frac": gbs / hbm_peak(),
                                 "what": "fks_moments (a10, 8 B read per phase-space point), HBM-bound"}
        ctx.check()
        if c["dx_dim"] == 0 and dv == 3 and not a.no_spatial_secondary:
            extra["C4_fused_step"] = spatial_secondary("C4", stream, reps)
            extra["N64_step"] = n64_secondary(c["L"], A, c["tau"], dt, stream, reps)

    # ---- e2e through the C ABI with host buffers (H2D + step + D2H per step) --------------
    e2e = None
    state_bytes = ncells * n * 8
    if not a.no_e2e and F is None and stepper is None and c["dx_dim"] > 0 and state_bytes <= (8 << 30):
        F = fa.cpu().numpy()  # the spatial configs' state, for the host-buffer path
    if not a.no_e2e and F is None and c["dx_dim"] > 0:
        e2e = {"value": None, "unit": "cells/s",
               "why": f"state of {state_bytes / 2**30:.1f} GiB per copy: pinned host buffers not allocated (limit 8 GiB)"}
    if not a.no_e2e and F is not None and stepper is None:
        hin = torch.from_numpy(np.ascontiguousarray(F)).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        if c["dx_dim"] == 0:
            ctx_h = fks.Context(dv, 0, [ncells], N, c["L"], A)
        else:
            ctx_h = fks.Context(dv, c["dx_dim"], list(slab.M_local), N, c["L"], A, h=c["dx"], bc=slab.local_bc(c["bc"]))
            for face, g in workloads.ghost_vectors(c).items():
                ctx_h.set_ghost(face, torch.from_numpy(g).cuda())
            if sl is not None:
                ctx_h.set_solid(sl)
        ctx_h.set_params(tau=c["tau"])
        ctx_h.set_stream(stream)
        ctx_h.step_host(hin, hout, dt)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        ksteps = max(1, min(a.steps, 5))
        for _ in range(ksteps):
            ctx_h.step_host(hin, hout, dt)
            hin, hout = hout, hin
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        bytes_ = ncells * n * 8
        e2e = {"value": nfluid_local * world * ksteps / el, "unit": "cells/s", "h2d_bytes_per_step": bytes_,
               "d2h_bytes_per_step": bytes_, "steps": ksteps, "path": "fks_step_host (pinned host buffers)"}
        ctx_h.close()

    traffic, traffic_src = dram_traffic(dv, nfluid_local, a.config)
    if rank == 0:
        cpu = None
        if not a.no_cpu_baseline and world == 1:
            rate, cores, tot, wall = oracle_rate(a.config, seconds=15.0)
            cpu = {"value": rate, "unit": "cells/s", "cores": cores, "kind": "oracle",
                   "sample": f"{tot} cells of {a.config} (oracle collide_fft + projection + Euler, numpy fp64) "
                             f"in {wall:.1f} s on {cores} single-threaded processes"}
            try:
                cpu["direct"] = direct_timing()
            except MemoryError:
                cpu["direct"] = None
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.config}: " + {
                "C1": "0Dx2D BKW ensemble, Maxwell molecules, Nv=32^2, A=8",
                "C2": "0Dx3D two-Gaussian relaxation ensemble (Test 1.3 shape), hard spheres, Nv=32^3, "
                      "A=24 spherical 7-design",
                "C3": "1Dx3D Sod shock tube (Test 2.3 shape), 400 cells, Dirichlet ghosts, hard spheres, Nv=32^3, A=24",
                "C4": "2Dx3D re-entry geometry (Test 3.2 boxes), 100^2 cells, inflow/outflow, solids frozen, "
                      "hard spheres, Nv=32^3, A=24",
                "C5": "3Dx3D re-entry (Test 4.1), 48^3 cells with a 12^3 solid cuboid, inflow/outflow, "
                      "hard spheres, Nv=32^3, A=24"}.get(a.config, a.config),
                "cells_per_gpu": ncells, "fluid_cells_total": nfluid, "Nv": N, "dv": dv, "M_dirs": A, "dt": dt,
                "l2": f"inputs larger than L2 ({2 * ncells * n * 8 / 2**30:.2f} GiB ping-pong state)"
                      if 2 * ncells * n * 8 > 126e6 else "state smaller than L2 (not flushed)",
                "parallelism": (f"dp{world} (independent cells, no collective)" if c["dx_dim"] == 0 else
                                f"{world} slabs along space axis {c['dx_dim'] - 1}, NCCL halo exchange per step")},
            "phase_space_updates_per_s": value * n,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "traffic_unit": f"bytes per launch (ncu dram read+write per cell x cells, {traffic_src})",
                         "peak_source": FP64_PEAK_SOURCE,
                         "algorithmic_bytes": 2 * n * 8 * ncells,
                         "hbm_frac": (2 * n * 8 * nfluid_local / (kern_avg_ms * 1e-3) / 1e9) / hbm_peak(),
                         "kernel": "k_step3d" if dv == 3 else "k_step2d",
                         "flops_per_cell": fl, "kernel_ms_avg": kern_avg_ms,
                         "note": "flops in the 5 n log2 n FFT convention (SURVEY App. A.9); the peak is the "
                                 "sustained DFMA measurement when profiles/r02_peaks.json holds one"},
            "gpu_launches": launches,
            "secondary": extra,
            "clocks": clk,
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
