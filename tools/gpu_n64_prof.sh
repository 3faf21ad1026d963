#!/bin/bash
# ncu --set full of one k_step3d64 launch (3D N = 64, 64 cells), summarised on the box.
cd "$(dirname "$0")/.."
O=gpurun_out/p64
mkdir -p $O
cat > $O/one.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, workloads
from paper_1608_08009_b200 import fks
N, L, nc = 64, 7.0, int(sys.argv[1])
f = workloads.family("smooth", 3, N, L, 8, seed=5)
F = torch.from_numpy(f).cuda().repeat((nc + 7) // 8, 1, 1, 1)[:nc].contiguous()
out = torch.empty_like(F)
ctx = fks.Context(3, 0, [nc], N, L, 24)
for _ in range(2):
    ctx.step(F, out, 0.01)
torch.cuda.synchronize()
ctx.check()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step3d64 --launch-skip 1 -c 1 -f -o $O/ncu_n64 python $O/one.py ${1:-64} > $O/ncu_n64.log 2>&1
python tools/ncu_summary.py $O/ncu_n64.ncu-rep k_step3d64 ${1:-64} $O/ncu_n64.json "ncu --set full --clock-control none, 3D N=64" > $O/ncu_n64.summary.txt 2>&1
ncu -i $O/ncu_n64.ncu-rep --page raw --csv > $O/ncu_n64.raw.csv 2>/dev/null
ncu -i $O/ncu_n64.ncu-rep --page source --csv --print-source sass > $O/ncu_n64.sass.csv 2>/dev/null
ncu -i $O/ncu_n64.ncu-rep --page details --csv > $O/ncu_n64.details.csv 2>/dev/null
rm -f $O/ncu_n64.ncu-rep
