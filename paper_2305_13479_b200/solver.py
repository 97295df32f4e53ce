"""Solver interface: the `pdlp-b200` backend behind the reference's API.

Mirrors collsched.solver (pkg/src/collsched/solver.py:30-169): same option
and solution types, same status names, same `solve(m, opts)` and
`min_feasible_horizon` entry points. The only backend is the GPU PDLP
engine in libteccl_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native as nat
from .errors import HorizonInfeasibleError, SolverBackendError, ValidationError
from .lp import DeviceLP

OPTIMAL = "optimal"
FEASIBLE_GAP = "feasible-gap"
INFEASIBLE = "infeasible"
TIMEOUT = "timeout"

ENV_BACKEND = "COLLSCHED_SOLVER"
BACKEND = "pdlp-b200"


@dataclass(frozen=True)
class SolverOptions:
    time_limit: float = 300.0
    relative_gap: float = 0.0          # reference meaning (MIP gap); LPs ignore it
    seed: int = 0
    verbosity: int = 0
    backend: str | None = None         # None: $COLLSCHED_SOLVER or "pdlp-b200"
    eps_rel: float = 1e-4              # PDLP relative KKT tolerance
    max_iters: int = 2_000_000
    check_every: int = 64
    device: int = 0
    pdlp: dict = field(default_factory=dict)   # raw teccl_pdlp_opts overrides (tuning)

    def __post_init__(self):
        if not (0 <= self.relative_gap < 1):
            raise ValidationError("relative_gap must be in [0, 1)")
        if self.time_limit <= 0:
            raise ValidationError("time_limit must be positive")
        if not self.eps_rel > 0:
            raise ValidationError("eps_rel must be positive")


@dataclass
class Solution:
    status: str
    model: object
    x: np.ndarray | None = None
    objective: float | None = None     # maximisation sense, like the reference
    achieved_gap: float = 0.0
    solve_wall_time: float = 0.0
    meta: dict = field(default_factory=dict)
    y: np.ndarray | None = None

    @property
    def feasible(self) -> bool:
        return self.status in (OPTIMAL, FEASIBLE_GAP)


def _backend_name(opts: SolverOptions) -> str:
    return opts.backend or os.environ.get(ENV_BACKEND, BACKEND)


def pdlp_options(opts: SolverOptions, verbose: int = 0) -> nat.PdlpOpts:
    o = nat.PdlpOpts()
    nat.load().teccl_pdlp_default_opts(C.byref(o))
    o.eps_rel = float(opts.eps_rel)
    o.max_iters = int(opts.max_iters)
    o.time_limit = float(opts.time_limit)
    o.check_every = int(opts.check_every)
    o.verbose = int(verbose)
    for k, v in opts.pdlp.items():
        setattr(o, k, type(getattr(o, k))(v))
    return o


def _upload_generic(m, device: int) -> DeviceLP:
    """Reference-style Model (num_vars, kinds, lb, ub, rows, objective) ->
    device LP, minimisation form c = -objective (solver.py:96-118)."""
    ctx = nat.Context.get(device)
    n = m.num_vars
    c = np.zeros(n)
    for idx, coef in m.objective.items():
        c[idx] = -coef
    lb = np.asarray(m.lb, dtype=np.float64)
    ub = np.array([np.inf if b == float("inf") else b for b in m.ub], dtype=np.float64)
    rp = np.zeros(len(m.rows) + 1, np.int64)
    cols, vals, lo, hi = [], [], [], []
    for r, (coeffs, rlo, rhi) in enumerate(m.rows):
        for idx, coef in coeffs:
            cols.append(idx)
            vals.append(coef)
        rp[r + 1] = len(cols)
        lo.append(-np.inf if rlo == -float("inf") else rlo)
        hi.append(np.inf if rhi == float("inf") else rhi)
    col = np.asarray(cols, np.int32)
    val = np.asarray(vals, np.float64)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    h = C.c_void_p()
    nat.check(ctx.lib.teccl_lp_from_csr(
        ctx.handle, len(m.rows), n, len(cols), nat.ptr(rp, C.c_int64), nat.ptr(col, C.c_int32),
        nat.ptr(val, C.c_double), nat.ptr(lo, C.c_double), nat.ptr(hi, C.c_double),
        nat.ptr(lb, C.c_double), nat.ptr(ub, C.c_double), nat.ptr(c, C.c_double), C.byref(h)))
    return DeviceLP(h, ctx, None, name=getattr(m, "name", "model"))


def solve(m, opts: SolverOptions | None = None, relax_integrality: bool = False,
          verbose: int = 0, warm: Solution | None = None) -> Solution:
    """Solve an LP on the GPU. `m` is a DeviceLP (from build_lp_model) or any
    reference-style Model whose variables are all continuous. `warm`: a
    previous Solution of the same LP (x and y) to start the iteration from."""
    opts = opts or SolverOptions()
    name = _backend_name(opts)
    if name != BACKEND:
        raise SolverBackendError(f"unknown solver backend {name!r} (available: {BACKEND})")
    dev_lp = m if isinstance(m, DeviceLP) else None
    if dev_lp is None:
        kinds = getattr(m, "kinds", [])
        if not relax_integrality and any(k in ("B", "I") for k in kinds):
            raise SolverBackendError(
                "pdlp-b200 solves linear programs; pass relax_integrality=True for a relaxation")
        if m.num_vars == 0:
            return Solution(OPTIMAL, m, np.zeros(0), 0.0)
        dev_lp = _upload_generic(m, opts.device)
    t0 = time.perf_counter()
    x = np.empty(dev_lp.num_vars)
    y = np.empty(dev_lp.num_rows)
    res = nat.PdlpResult()
    o = pdlp_options(opts, verbose)
    if warm is not None:
        if warm.x is None or warm.y is None or len(warm.x) != len(x) or len(warm.y) != len(y):
            raise ValidationError("warm start needs x and y of this LP")
        x[:] = warm.x
        y[:] = warm.y
        o.warm_start = 1
    nat.check(dev_lp.ctx.lib.teccl_pdlp_solve(dev_lp.ctx.handle, dev_lp.handle, C.byref(o),
                                              nat.ptr(x, C.c_double), nat.ptr(y, C.c_double),
                                              C.byref(res)))
    wall = time.perf_counter() - t0
    st = nat.STATUS.get(res.status, "numerical")
    status = {"optimal": OPTIMAL, "iteration-limit": TIMEOUT, "time-limit": TIMEOUT,
              "primal-infeasible": INFEASIBLE}.get(st, TIMEOUT)
    meta = {"iters": int(res.iters), "restarts": int(res.restarts),
            "rel_primal_res": res.rel_primal_res, "rel_dual_res": res.rel_dual_res,
            "rel_gap": res.rel_gap, "dual_objective": -res.dual_obj,
            "device_seconds": res.solve_seconds, "pdlp_status": st, "step": res.step,
            "omega": res.omega, "kernel_launches": int(res.spmv_launches),
            "eps_rel": opts.eps_rel}
    return Solution(status, m, x, float(-res.primal_obj), float(res.rel_gap), wall, meta, y)


def min_feasible_horizon(builder: Callable[[int], object], k_lo: int, k_hi: int,
                         opts: SolverOptions | None = None) -> tuple[int, Solution]:
    """Binary search of the smallest feasible horizon (solver.py:140-169).

    A first-order method cannot certify infeasibility by itself; for models
    from build_lp_model every probe first solves the phase-1 LP
    (lp.feasibility_gap), exactly like the reference's HiGHS infeasible
    status drives its search."""
    if k_lo < 1 or k_hi < k_lo:
        raise ValidationError(f"bad horizon range [{k_lo}, {k_hi}]")
    from .lp import horizon_feasible
    best = None
    lo, hi = k_lo, k_hi
    while lo <= hi:
        mid = (lo + hi) // 2
        m = builder(mid)
        plan = getattr(m, "plan", None)
        if plan is not None:
            # time-expanded model: certify (in)feasibility with the phase-1 LP,
            # then solve the real LP only at feasible horizons
            ok = horizon_feasible(plan, getattr(m.ctx, "device", 0))
            sol = solve(m, opts) if ok else Solution(INFEASIBLE, m)
        else:
            sol = solve(m, opts)
        if sol.feasible:
            best = (mid, sol)
            hi = mid - 1
        else:
            lo = mid + 1
    if best is None:
        raise HorizonInfeasibleError(k_lo, k_hi)
    return best
