"""CPU oracle for arXiv 2405.18982 (Cui & Kanschat, *Multilevel Interior Penalty
Methods on GPUs*) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct fp64 (optionally fp32) CPU
implementation of what the GPU hot path computes:

* ``basis``     -- GLL Lagrange basis and Gauss quadrature (App. A)
* ``mesh``      -- Cartesian hierarchy, cell-wise lexicographic numbering, vertex
                   patches and their 2^d colours
* ``assemble``  -- element-by-element quadrature assembly of the SIPG matrix
                   (eq. bilinear_form) into CSR, and the RHS
* ``transfer``  -- canonical-embedding prolongation and its transpose
* ``smoother``  -- colourised multiplicative / additive vertex-patch Schwarz
                   smoother with *dense LU* local solves of A_j = R_j A R_j^T
                   extracted from the assembled matrix (Alg. 1)
* ``multigrid`` -- the V-cycle of PAPER.md:155-172 with a dense coarse solve
* ``krylov``    -- PCG, right-preconditioned GMRES, fractional iteration count nu
                   

Rules: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2405_18982_b200`` (the CUDA path) and
never imports it; the only common module is ``synth_inputs`` (seeded random
inputs, no method arithmetic).

Parity status: every public function is pinned by ``tests/test_oracle_*.py``
against values the paper/SPEC print, closed forms, or brute-force checks.
"""
