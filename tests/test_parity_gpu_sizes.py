"""Large and ragged cell counts on the kernels added last (64^3, N = 4, 2D N = 64): many rounds of
the persistent grids, the last one partial, checked on sampled cells against the oracle (the
FFT evaluator, itself pinned to the literal sum) -- SURVEY §8(c.5) 'at sizes that span several
tiles and a ragged tail'."""
import numpy as np
import pytest

import workloads
from oracle import step as ostep, tables

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    if not _t.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return _t


@pytest.mark.parametrize("dv,N,L,A,nc,sample", [
    (3, 64, 7.0, 24, 301, [0, 3, 150, 299, 300]),          # 4 groups: 76 rounds, the last with one cell
    (3, 4, 4.0, 24, 10007, [0, 1, 4735, 4736, 10006]),     # 4 cells per CTA, 1184 CTAs per round
    (2, 4, 3.0, 8, 100003, [0, 17, 18943, 18944, 100002]),  # 16 cells per CTA
    (2, 64, 12.0, 8, 40001, [0, 295, 296, 40000]),          # 2 cells per CTA, 148 CTAs
])
def test_many_cells_sampled(torch, dv, N, L, A, nc, sample):
    from paper_1608_08009_b200 import fks
    base = workloads.family("smooth", dv, N, L, 7, seed=nc % 97)
    scale = 0.5 + np.arange(nc) % 13 / 13.0
    idx = np.arange(nc) % 7
    F = torch.from_numpy(base).cuda()[torch.from_numpy(idx).cuda()] * torch.from_numpy(scale).cuda().view(
        (nc,) + (1,) * dv)
    ctx = fks.Context(dv, 0, [nc], N, L, A)
    ctx.set_params(tau=0.6)
    out = torch.empty_like(F)
    dt = 0.05
    ctx.step(F, out, dt)
    ctx.check()
    tab = tables.build_tables(2, N, L, A=A) if dv == 2 else tables.build_tables(3, N, L)
    got = out[sample].cpu().numpy()
    fin = np.stack([base[idx[c]] * scale[c] for c in sample])
    ref = ostep.homogeneous_step(fin, tab, dt, tau=0.6)
    for i in range(len(sample)):
        assert np.max(np.abs(got[i] - ref[i])) <= TOL * np.max(np.abs(ref[i])), sample[i]
