"""fks_step_host end-to-end rate on C2 (4096 cells) for the FKS_HOST_CHUNKS values given on the
command line (development aid; each value in a fresh context, 5 timed steps after 2 warm-ups)."""
import os
import subprocess
import sys

CODE = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, workloads
from paper_1608_08009_b200 import fks
c = workloads.config("C2"); N, L = c["N"], c["L"]; nc = 4096
base = workloads.initial_state(c, ncells=256)
F = np.concatenate([base] * 16)
hin = torch.from_numpy(F).pin_memory(); hout = torch.empty_like(hin).pin_memory()
ctx = fks.Context(3, 0, [nc], N, L, 24)
for _ in range(2):
    ctx.step_host(hin, hout, c["dt"])
t0 = time.perf_counter()
for _ in range(5):
    ctx.step_host(hin, hout, c["dt"]); hin, hout = hout, hin
el = time.perf_counter() - t0
print(os.environ.get("FKS_HOST_CHUNKS"), "chunks:", f"{5 * nc / el:.4g} cells/s", f"{el / 5 * 1e3:.2f} ms/step")
'''
for v in sys.argv[1:]:
    env = dict(os.environ, FKS_HOST_CHUNKS=v)
    subprocess.run([sys.executable, "-c", CODE], env=env)
