"""CPU oracle for arXiv 2404.10221 -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct CPU (numpy, FP64; setup tables
in x86 80-bit long double) implementation of what the tau-preconditioned GMRES
hot path computes, written from PAPER.md.  It is the yardstick the CUDA library
is checked against.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it; the
product path (``paper_2404_10221_b200``) never does, and it shares no code with
the CUDA path (the only shared module is ``paper_2404_10221_b200.inputs``, which
holds problem data and seeded generators, none of the method's arithmetic).

Modules:
  fcd     -- FCD generator, H_alpha, Toeplitz/Hankel, tau(T), q, DST-I (1-D)
  dense   -- Tier D: dense Kronecker assembly in the paper's order (N^d <= ~4096)
  lines   -- Tier L: per-line operators on grid arrays (dense n x n per axis)
  gmres   -- textbook restarted GMRES (MGS Arnoldi + Givens)
  scheme  -- RHS F, e-bar, preconditioner spectra, the CN time loop

Parity status: every function is pinned by tests/test_oracle_*.py against a
value the paper prints, a closed form, an invariant, a brute-force dense
computation or an independent library routine; see DESIGN.md "Oracle pins".
Nothing here is "parity unpinned".
"""
