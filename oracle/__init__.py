"""CPU oracle for the FE-evaluation hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain numpy/scipy restatement of the reference package's
(`romtopt`, /root/reference/pkg/src/romtopt) algorithm for the hot path named
by BASELINE.json's north_star:

    psi -(Helmholtz filter)-> rho -> K(rho) u = f -> compliance, per-element
    sensitivity -> filter adjoint;  Phi^T f, Phi^T K(rho) Phi, reduced solve,
    ||K(rho) Phi y - f||.

Every function cites the reference file:line it restates.  The 2D path is
pinned against golden vectors produced by running the reference itself in the
build container (tests/golden/make_golden.py -> tests/golden/*.npz).  The 3D
(Hex8) path has no reference implementation (the reference is 2D only,
SPEC.md:18); it follows the reference's dimension-generic routines
(hdm.py:211-233, rom.py:254-325) and the reference's own quadrature oracles
(tests/oracles.py:44-89), and is pinned by the reference's HdmSolver/RomModel
run on a duck-typed 3D mesh (golden file ``ref3d_*.npz``) plus the
dimension-independent filter identities (volume preservation, constant
preservation, exact transpose).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU reference arm.  The product package ``paper_2004_05756_b200``
never imports it.
"""
