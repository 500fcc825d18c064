"""CPU oracle for the PinT QBVM/MQBVM hot path -- TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it. The product package
(``paper_2107_06381_b200``) never imports anything from here and has no CPU
fallback: without its CUDA library it raises.

Contents (each function cites the reference file:line it restates; paths are
relative to the reference checkout ``pkg/src/bhcp``):

* ``bhcp_oracle`` -- numpy restatement of the reference algorithm: time grid,
  omega/divisor, Gamma/eigenvalue diagonalisation, time transforms, DST-I,
  Laplacian spectrum (extended to 3D), shifted solves, the 3-step
  ``solve_pint`` and the closed-form spectral oracle, plus the seeded
  BASELINE.json workload generators.

Parity pinning: the restatement is checked against golden vectors produced by
running the *reference itself* (``tests/golden/make_golden.py`` imports the
read-only reference package and writes ``tests/golden/*.npz``) and against the
known-answer tests of the reference test-suite (closed forms). The 3D
extension has no reference counterpart (the reference rejects dim=3,
space.py:42-43); it is pinned by separable-mode reductions to the 1D/2D
golden cases.
"""
