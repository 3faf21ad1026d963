"""CPU oracle for the FKS + fast-spectral Boltzmann hot path (arXiv 1608.08009).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_1608_08009_b200``) never imports it
and never falls back to it.

The oracle is a plain, slow, fp64 numpy implementation written from the paper.
It shares no code with the CUDA path: no kernels, headers, tables, constants or
helpers.  The only thing both sides consume is the bytes produced by the seeded
input generators in ``workloads/`` (which hold none of the method's arithmetic).

Citation keys: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line
n; "reading #k" = the k-th entry of DESIGN.md §"Readings of the paper".

Modules
-------
grid        velocity lattice, mode numbers, mirror map
kernels     radial functions phi, phi3, psi3 and direction sets
tables      alpha, alpha', D tables (symmetrised)
collision   direct O(n^2) bilinear form and the cpu_fft evaluator
projection  L2 conservation projection
transport   FKS shift tables and the boundary-aware gather
step        first-order split step
moments     rho, u, T
brute       sigma-representation quadrature of Q_B
bkw         BKW exact solution

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against closed forms, printed values of the paper,
brute force or invariants; see DESIGN.md §"Oracle pins".
"""
