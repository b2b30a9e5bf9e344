"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU implementation of the
SIPDG Poisson operator and the conjugate-gradient solve of Karakus et al.,
arXiv:1801.00246 ("PAPER.md" below; P:n = line n of PAPER.md).  It exists only
to prove the CUDA path right.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.  The
product package ``paper_1801_00246_b200`` never imports it, and it never
imports the product package: the two share no code.  Inputs (meshes, random
fields) come from ``paper_1801_00246_b200.meshgen``, a module that holds none of
the method's arithmetic; the tests hand them to both sides.

All arithmetic is numpy/scipy float64 (the paper computes in double precision,
P:384), plus exact rationals (``fractions.Fraction``) in ``oracle.exact``.

Modules (each function cites the passage it follows):
  refelem     reference triangle: Warp & Blend nodes, PKD basis, Dr, Ds, M, LIFT
  quadrature  Gauss-Jacobi / Gauss-Lobatto rules, collapsed triangle rule
  meshops     connectivity by coordinate matching, affine geometry, penalty tau
  assemble    SIPDG bilinear form (Eq. ellipticOp1) assembled by quadrature -> CSR
  exact       the same bilinear form in exact rational arithmetic (N <= 2)
  mfree       matrix-free primal face loop (numpy, for timing at scale)
  solvers     textbook (P)CG and the manufactured right-hand side

Parity-pin status: every function here is pinned by tests/test_oracle_*.py
against closed forms, paper values, exact rationals or brute force; none is
"parity unpinned" (see DESIGN.md section "Oracle pins").
"""
