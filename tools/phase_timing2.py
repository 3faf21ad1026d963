"""Per-direction phase stamps (clock64) of group 0 / CTA 0, warp 0 of each warp group, on the
group's third cell (steady state), C2 shape.  Build: FKS_TIMING=1 python -m paper_1608_08009_b200.build;
run with FKS_LIB_VARIANT=timing (development aid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1608_08009_b200 import _lib, fks  # noqa: E402

c = workloads.config("C2")
N, L = c["N"], c["L"]
nc = 144
f = workloads.initial_state(c, ncells=48)
F = np.concatenate([f] * 3)
ctx = fks.Context(3, 0, [nc], N, L, 24)
a = torch.from_numpy(F).cuda()
b = torch.empty_like(a)
for _ in range(2):
    ctx.step(a, b, c["dt"])
    torch.cuda.synchronize()
buf = (ctypes.c_longlong * 4096)()
_lib.load().fks_debug_tstamps(buf, 4096)
ts = np.array(buf[:])
base = ts[0]
r = lambda v: (v - base) if v else -1  # noqa: E731
print("d | xy: top landed xdone ydone | dur land x y | z: top tland zcomp stored | dur tw comp st")
for d in range(26):
    xy = [r(v) for v in ts[d * 8:d * 8 + 4]]
    z = [r(v) for v in ts[2048 + d * 8:2048 + d * 8 + 4]]
    nxt = r(ts[(d + 1) * 8]) if d < 25 else -1
    nz = r(ts[2048 + (d + 1) * 8]) if d < 25 else -1
    print(f"{d:2d} | " + " ".join(f"{v:7d}" for v in xy) + f" | {nxt - xy[0]:5d} {xy[1]-xy[0]:5d} {xy[2]-xy[1]:5d} {xy[3]-xy[2]:5d} | "
          + " ".join(f"{v:7d}" for v in z) + f" | {nz - z[0]:5d} {z[1]-z[0]:5d} {z[2]-z[1]:5d} {z[3]-z[2]:5d}")
