"""Launch one hot-path call of a BASELINE config in bench.py's configuration, for ncu / compute-sanitizer
captures (development aid; bench.py is the contract):

  python tools/profile_launch.py C4 step [reps] [--small]

what: step | collide | transport | moments | bgk.  --small shrinks the workload (sanitizer runs).
The first call is a warm-up; `reps` more calls follow (capture them with ncu --launch-skip).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1608_08009_b200 import fks  # noqa: E402


def main():
    name, what = sys.argv[1], sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 1
    small = "--small" in sys.argv
    c = workloads.config(name)
    dv, N, A = c["dv"], c["N"], c["A"]
    n = N ** dv
    if c["dx_dim"] == 0:
        nc = (37 if small else c["cells"][0])
        base = workloads.initial_state(c, ncells=min(nc, 64))
        F = np.concatenate([base] * ((nc + base.shape[0] - 1) // base.shape[0]))[:nc]
        ctx = fks.Context(dv, 0, [nc], N, c["L"], A)
        fa = torch.from_numpy(F.reshape(nc, -1)).cuda()
    else:
        M = list(c["cells"][::-1])
        if small:
            M = [min(m, 6) for m in M]
        ctx = fks.Context(dv, c["dx_dim"], M, N, c["L"], A, h=c["dx"], bc=c["bc"])
        for face, g in workloads.ghost_vectors(c).items():
            ctx.set_ghost(face, torch.from_numpy(g).cuda())
        solid = workloads.solid_mask(c)
        if solid is not None and not small:
            ctx.set_solid(solid)
        nc = int(np.prod(M))
        v = torch.from_numpy(workloads.initial_state(c, ncells=1).reshape(-1)[:n].copy()).cuda()
        s = torch.from_numpy(1.0 + 0.1 * np.random.default_rng(1).random(nc)).cuda()
        fa = (v[None, :] * s[:, None]).contiguous()
    ctx.set_params(tau=c["tau"])
    fb = torch.empty_like(fa)
    rho = torch.empty(nc, dtype=torch.float64, device="cuda")
    u = torch.empty(nc, dv, dtype=torch.float64, device="cuda")
    T = torch.empty(nc, dtype=torch.float64, device="cuda")
    calls = {
        "step": lambda: ctx.step(fa, fb, c["dt"]),
        "collide": lambda: ctx.collide(fa, fb),
        "transport": lambda: ctx.transport(fa, fb, c["dt"]),
        "moments": lambda: ctx.moments(fa, rho, u, T),
        "bgk": lambda: ctx.step_bgk(fa, fb, c["dt"], fks.NU_RHO, 0.0),
    }
    for _ in range(1 + reps):
        calls[what]()
    ctx.check()
    torch.cuda.synchronize()
    print(f"{name} {what}: {nc} cells, {1 + reps} calls ok")


if __name__ == "__main__":
    main()
