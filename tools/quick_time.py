"""Quick CUDA-event timing of fks_step on C1/C2 (development aid; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
from paper_1608_08009_b200 import fks

def run(name, ncells=None, steps=5):
    c = workloads.config(name)
    nc = ncells or c["cells"][0]
    N, L, dv = c["N"], c["L"], c["dv"]
    f = workloads.initial_state(c, ncells=min(nc, 64))
    reps = (nc + f.shape[0] - 1) // f.shape[0]
    F = np.concatenate([f] * reps)[:nc]
    ctx = fks.Context(dv, 0, [nc], N, L, c["A"])
    a = torch.from_numpy(F).cuda(); b = torch.empty_like(a)
    for _ in range(2):
        ctx.step(a, b, c["dt"]); a, b = b, a
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        ctx.step(a, b, c["dt"]); a, b = b, a
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.check()
    print(f"{name}: {nc} cells, {ms:.3f} ms/step, {nc/ms*1e3:.4g} cells/s, {nc*N**dv/ms*1e3:.4g} updates/s")

run("C1", steps=10)
run("C2", steps=3)
from paper_1608_08009_b200 import _lib
