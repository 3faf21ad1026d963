"""Read the per-phase clock64 stamps of cluster 0 / CTA 0 (build with FKS_TIMING=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
from paper_1608_08009_b200 import fks, _lib
c = workloads.config("C2")
N, L = c["N"], c["L"]
nc = 256
f = workloads.initial_state(c, ncells=64)
F = np.concatenate([f] * 4)
ctx = fks.Context(3, 0, [nc], N, L, 24)
a = torch.from_numpy(F).cuda(); b = torch.empty_like(a)
ctx.step(a, b, c["dt"]); torch.cuda.synchronize()
ctx.step(b, a, c["dt"]); torch.cuda.synchronize()
buf = (ctypes.c_longlong * 4096)()
_lib.load().fks_debug_tstamps(buf, 4096)
ts = np.array(buf[:])
base = ts[2 * 8]
def r(v): return v - base if v else -1
print("k | xy: top  Wland  xdone  ydone  arrive  waitret  issued | z: top acq released stored waitret computed barred")
for k in range(27):
    xy = [r(v) for v in ts[k*8:k*8+7]]
    z = [r(v) for v in ts[2048+k*8:2048+k*8+7]]
    print(k, "|", " ".join(f"{v:7d}" for v in xy), "|", " ".join(f"{v:7d}" for v in z))
if ts[1024]:
    print("chunk consume: t0 | wait  lds+st  bar  issue (cycles)")
    for g in range(64):
        v = ts[1024 + g * 8:1024 + g * 8 + 5]
        if v[0]:
            print(g, v[0] - base, "|", " ".join(f"{v[i+1]-v[i]:6d}" for i in range(4)))
if ts[3072 + 8]:
    print("table slab g (cp_thr: wait-tbar start, landed, cp issued | ld_thr: wait-tcp start, cp done)")
    for g in range(1, 40):
        v = ts[3072 + g * 8:3072 + g * 8 + 8]
        if v[0] or v[3]:
            print(g, " ".join(f"{(x - base) if x else -1:7d}" for x in v))
names = ["z fwd start", "z fwd rows done", "z fwd W stored+signalled", "xy cell start (load z(0))", "xy epilogue start",
         "xy partials ready", "xy lambda ready", "xy cell done", "-", "z fwd available", "z fwd read+FFT done"]
print("cell boundary (cell 0 epilogue = first set; cell 1 forward = second set)")
for c in range(2):
    for i, nm in enumerate(names):
        v = ts[1024 + c * 16 + i]
        if v:
            print(f"  cell{c} {nm:24s} {v - base:8d}")
# per-rank global timer (ns) of group 0: xy direction tops, epilogue, z stores done
buf2 = (ctypes.c_longlong * 4096)()
_lib.load().fks_debug_tstamps(buf2, 4096)
g = np.array(buf2[:])[3072:3072 + 8 * 128].reshape(8, 128)
t0 = g[:, 0].min()
print("rank | xy top d=0,5,10,15,20,24 (cell0, us) | epi start, lambda (cell0) | z stored j=23 cell0 | xy top d=0 cell1")
for r in range(8):
    row = g[r]
    f = lambda v: f"{(v - t0) / 1000:7.2f}" if v else "   -   "
    print(r, "|", " ".join(f(row[d]) for d in (0, 5, 10, 15, 20, 24)), "|", f(row[30]), f(row[31]), "|", f(row[80 + 23]), "|", f(row[40]))
