"""CPU ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 CPU implementation of the stress-velocity
(primal-dual) Newton step of Shih, Mehlmann, Losch & Stadler (arXiv 2204.10822,
`/root/reference/PAPER.md`, cited as P:<line>).  It shares no code with the
CUDA path (`paper_2204_10822_b200/csrc`): it is written in the paper's 2x2
tensor notation (tau, pi as matrices, ":" the Frobenius product), while the
kernels use an orthonormal 3-vector basis.  Only `paper_2204_10822_b200.workloads`
(seeded input generation, no method arithmetic) is imported by both.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  The product path never does.

Parity status per function (see DESIGN.md §13 "Oracle pins"):
  fem.*            pinned (closed-form Q1 tables, mass matrix, quadrature exactness)
  model.residual   pinned (Phi' = -R by FD; worked example; vanishing cases)
  model.energy /
  model.delta_energy   pinned (FD, convexity, direct difference at large steps)
  model.jacobian   pinned (std: central FD of R; sv == std at consistent pi;
                   sv == sym(K) for s = 1; SPD; rigid-body nullspace)
  model.pi_tilde   pinned (FD of tau/Delta at consistent pi; closed forms)
  newton.solve_step  pinned (quadratic tail; manufactured solution rate;
                   yield-curve bound; direct vs Krylov solutions)
  krylov.*         pinned (textbook cases, dense solve comparison)
  transport.*      pinned (zero velocity, textbook 1-D upwind, conservation, Q1 midpoint
                   face velocities, monotonicity / clamping; tests/test_oracle_transport.py)
  amg.*            pinned for the algebra (Galerkin identity, P_tent
                   orthonormality, near-nullspace reproduction, single-level
                   exactness, V-cycle symmetry, Chebyshev closed form, MIS(2)
                   validity, aggregate partition; tests/test_oracle_amg.py);
                   "parity unpinned" for the hierarchy SHAPE (levels, aggregate
                   counts) — the aggregation is a definition, not a paper result.
"""
