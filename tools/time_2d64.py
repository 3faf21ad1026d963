"""CUDA-event timing of the 2D N = 64 fused step (k_step2dp<64>) -- development aid."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1608_08009_b200 import fks  # noqa: E402

N, L, A = 64, 12.0, 8
nc = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
f = workloads.family("bkw", 2, N, L, 64, seed=5)
F = torch.from_numpy(f).cuda().repeat((nc + 63) // 64, 1, 1)[:nc].contiguous()
out = torch.empty_like(F)
ctx = fks.Context(2, 0, [nc], N, L, A)
n = N * N
fl = (A + 1) * 5 * n * math.log2(n) + (9 * A + 25) * n
for _ in range(2):
    ctx.step(F, out, 0.01)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    ctx.step(F, out, 0.01)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
ctx.check()
tf = fl * nc / (ms * 1e-3) / 1e12
print(f"2D N=64 A={A}: {nc} cells, {ms:.3f} ms/step, {nc / ms * 1e3:.4g} cells/s, {tf:.2f} TF/s = "
      f"{tf / 36.947:.3f} of the sustained FP64 peak")
