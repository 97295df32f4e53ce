"""Solver interface: the `pdlp-b200` backend behind the reference's API.

Mirrors collsched.solver (pkg/src/collsched/solver.py:30-169): same option
and solution types, same status names, same `solve(m, opts)` and
`min_feasible_horizon` entry points. The only backend is the GPU PDLP
engine in libteccl_b200.so; there is no CPU fallback.

Statuses follow the reference (solver.py:128-144): "optimal" when the
duality gap is within eps_rel and both residuals within min(eps_rel,
eps_res) -- the defaults are north_star's parity bar, gap 1e-4 and residuals
1e-6 --, "infeasible" when the device found a Farkas certificate
(teccl_pdlp_opts.eps_infeas; x is None, like the reference's), "timeout" on
the iteration / time cap. A numerical failure raises SolverBackendError, as
the reference does for an unexpected HiGHS status (solver.py:136-138).
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
    eps_rel: float = 1e-4              # PDLP relative duality-gap tolerance
    eps_res: float = 1e-6              # relative primal / dual residual tolerance (capped at eps_rel)
    eps_infeas: float = 1e-6           # infeasibility-certificate margin (0: never "infeasible")
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
        if self.eps_res < 0 or self.eps_infeas < 0:
            raise ValidationError("eps_res and eps_infeas must be >= 0")


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
    o.eps_res = float(opts.eps_res)
    o.eps_infeas = float(opts.eps_infeas)
    o.max_iters = int(opts.max_iters)
    o.time_limit = float(opts.time_limit)
    o.check_every = int(opts.check_every)
    o.verbose = int(verbose)
    for k, v in opts.pdlp.items():
        setattr(o, k, type(getattr(o, k))(v))
    return o


def _upload_generic(m, device: int) -> DeviceLP:
    """Reference-style Model (num_vars, kinds, lb, ub, rows, objective) ->
    device LP, minimisation form c = -objective (solver.py:100-121)."""
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


def _rebuild_te(m, device: int):
    """A reference Model made by collsched's build_lp_model (meta kind "lp",
    lp.py:40-45) is rebuilt on the device from the inputs it records -- the
    same columns, rows, bounds and costs (pinned bit for bit by the builder
    goldens) -- so it gets the matrix-free operator and the time-expanded
    implied bounds of the infeasibility certificate. None when the model is
    something else or its shape no longer matches (mutated after the build)."""
    from .lp import build_lp_model
    meta = getattr(m, "meta", None) or {}
    if meta.get("kind") != "lp" or not all(k in meta for k in ("topology", "demand", "cfg")):
        return None
    try:
        lp = build_lp_model(meta["topology"], meta["demand"], meta["cfg"], meta.get("opts"),
                            device=device)
    except Exception:
        return None
    rows = getattr(m, "rows", None)
    if lp.num_vars != m.num_vars or (rows is not None and lp.num_rows != len(rows)):
        lp.close()
        return None
    return lp


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
    owned = False
    if dev_lp is None:
        kinds = getattr(m, "kinds", [])
        if not relax_integrality and any(k in ("B", "I") for k in kinds):
            raise SolverBackendError(
                "pdlp-b200 solves linear programs; pass relax_integrality=True for a relaxation")
        if m.num_vars == 0:
            return Solution(OPTIMAL, m, np.zeros(0), 0.0)
        dev_lp = _rebuild_te(m, opts.device) or _upload_generic(m, opts.device)
        owned = True
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
    if owned:
        dev_lp.close()
    st = nat.STATUS.get(res.status, "numerical")
    if st in ("numerical", "peer-timeout"):
        raise SolverBackendError(f"solver failed: PDLP status {st} after {res.iters} iterations")
    status = {"optimal": OPTIMAL, "iteration-limit": TIMEOUT, "time-limit": TIMEOUT,
              "primal-infeasible": INFEASIBLE}[st]
    meta = {"iters": int(res.iters), "restarts": int(res.restarts),
            "rel_primal_res": res.rel_primal_res, "rel_dual_res": res.rel_dual_res,
            "rel_gap": res.rel_gap, "dual_objective": -res.dual_obj,
            "device_seconds": res.solve_seconds, "pdlp_status": st, "step": res.step,
            "omega": res.omega, "kernel_launches": int(res.spmv_launches),
            "eps_rel": opts.eps_rel, "eps_res": min(opts.eps_rel, opts.eps_res) if opts.eps_res > 0
            else opts.eps_rel, "infeas_cert": res.infeas_cert}
    if status == INFEASIBLE:  # like the reference: no values for an infeasible model
        return Solution(INFEASIBLE, m, solve_wall_time=wall, meta=meta)
    return Solution(status, m, x, float(-res.primal_obj), float(res.rel_gap), wall, meta, y)


def min_feasible_horizon(builder: Callable[[int], object], k_lo: int, k_hi: int,
                         opts: SolverOptions | None = None) -> tuple[int, Solution]:
    """Binary search of the smallest feasible horizon, as the reference's
    (solver.py:146-168): every probe is one solve; "infeasible" (the device's
    Farkas certificate) moves up, a feasible solve moves down, a timed-out
    probe raises SolverBackendError. Device LPs of discarded probes are freed
    before the next build."""
    if k_lo < 1 or k_hi < k_lo:
        raise ValidationError(f"bad horizon range [{k_lo}, {k_hi}]")
    best = None
    lo, hi = k_lo, k_hi
    while lo <= hi:
        mid = (lo + hi) // 2
        m = builder(mid)
        sol = solve(m, opts)
        if sol.status == TIMEOUT:
            _close(m)
            raise SolverBackendError(f"horizon probe timed out at K={mid}")
        if sol.feasible:
            if best is not None:
                _close(best[1].model)
            best = (mid, sol)
            hi = mid - 1
        else:
            _close(m)
            lo = mid + 1
    if best is None:
        raise HorizonInfeasibleError(k_lo, k_hi)
    return best


def _close(m) -> None:
    if isinstance(m, DeviceLP):
        m.close()
