"""The reference-side hook: what collsched.solver.solve runs
when its backend is "pdlp-b200".

`reference_solve(m, opts)` takes the reference's own Model and SolverOptions
(pkg/src/collsched/solver.py:30-44, model.py:17-86; duck-typed, nothing is
imported from collsched) and returns a Solution with the reference's fields
and statuses (solver.py:47-55, 128-144): "optimal" at north_star's parity bar
(duality gap 1e-4, residuals 1e-6), "infeasible" from the device's Farkas
certificate, "timeout" at the time limit. A Model built by
collsched.lp.build_lp_model is rebuilt on the device from its recorded
inputs (solver._rebuild_te); any other continuous Model is uploaded as CSR.
"""

from __future__ import annotations

from .solver import Solution, SolverOptions, solve

BACKEND = "pdlp-b200"


def reference_solve(m, opts=None, relax_integrality: bool = False, device: int = 0) -> Solution:
    """collsched.solver.solve(m, opts) on the GPU engine."""
    time_limit = float(getattr(opts, "time_limit", 300.0)) if opts is not None else 300.0
    verbose = 100 if opts is not None and getattr(opts, "verbosity", 0) > 1 else 0
    return solve(m, SolverOptions(time_limit=time_limit, device=device),
                 relax_integrality=relax_integrality, verbose=verbose)
