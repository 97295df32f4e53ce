"""End-to-end LP synthesis on the GPU: build, solve, decompose, replay.

Mirrors the reference's `synthesize(t, d, method="lp", ...)`
(pkg/src/collsched/workflow.py:37-113) for the copy-free LP path: epoch
duration from the topology, the time-expanded LP built and solved on the
device, the rates decomposed into per-chunk events (lp_rates_to_schedule),
and the emitted EVENT LIST replayed by the native event simulator
(simulate.simulate, the reference's simulator.py:58-235) before anything is
returned -- a schedule that fails its replay raises instead of being
returned, like the reference's `_checked_replay` (workflow.py:125-132). The
flows the events were peeled from are also replayed by the exact-integer GPU
checker.

Differences, all outside the tier's hot path: only method "lp" (the MILP
and A* paths are out of scope); with `epochs=None` the horizon comes from a
doubling search of LP solves, each answered "infeasible" by the device's
Farkas certificate or solved (the reference's estimator solves MILPs).
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

from .checker import check_lp_schedule
from .demand import Demand
from .epochs import FASTEST, EpochConfig, epoch_duration
from .errors import (HorizonInfeasibleError, SolverBackendError, SolverTimeoutError,
                     ValidationError)
from .lp import HYPER_EDGE, COPY, ModelOptions, build_from_plan, make_plan
from .schedule import Schedule, schedule_with_flows
from .simulate import SimOptions, SimReport, simulate
from .solver import INFEASIBLE, TIMEOUT, SolverOptions, min_feasible_horizon, solve
from .topology import Topology

METHODS = ("lp",)
OUT_OF_SCOPE = ("milp", "astar")


@dataclass
class SynthesisResult:
    """Same fields as the reference's SynthesisResult (workflow.py:23-35);
    `report` is the event replay's SimReport (simulator.py:42-55), `check`
    the exact-integer flow checker's CheckReport."""
    schedule: Schedule
    report: SimReport
    method: str
    status: str
    solver_wall_time: float
    total_wall_time: float
    objective: float | None
    achieved_gap: float
    epochs: int
    tau: float
    warnings: list[str] = field(default_factory=list)
    check: object = None


def feasible_horizon(t: Topology, d: Demand, cfg: EpochConfig, opts: ModelOptions,
                     k0: int = 8, k_max: int = 1 << 20, device: int = 0,
                     sopts: SolverOptions | None = None) -> tuple:
    """(K, solution) for the smallest K = k0 * 2^j whose LP is feasible. Each
    probe is one solve: "infeasible" (the device certificate) doubles K, a
    timed-out probe raises like the reference's (solver.py:160-161)."""
    sopts = sopts or SolverOptions(device=device)
    K = max(1, k0)
    while K <= k_max:
        lp = build_from_plan(make_plan(t, d, cfg.with_horizon(K), opts), device)
        sol = solve(lp, sopts)
        if sol.feasible:
            return K, sol
        lp.close()
        if sol.status == TIMEOUT:
            raise SolverBackendError(f"horizon probe timed out at K={K}")
        K *= 2
    raise HorizonInfeasibleError(k0, k_max)


def synthesize(t: Topology, d: Demand, method: str = "lp", *,
               switch_mode: str = COPY, buffer_limit: float | None = None,
               epoch_mode: str = FASTEST, em: int = 1,
               epochs: int | None = None, search_horizon: bool = False,
               gap: float = 0.0, time_limit: float = 300.0,
               eps_rel: float = 1e-4, device: int = 0,
               check_tol: float = 1e-5, **ignored) -> SynthesisResult:
    """Produce a schedule with the GPU LP engine and verify it by replay.
    `gap` is the reference's MILP gap (unused by the LP); `eps_rel` is the
    PDLP gap tolerance (residuals to 1e-6); MILP / A* keywords (gamma,
    epochs_per_round, max_rounds, seed, dump_model_path) are accepted and
    ignored."""
    if method in OUT_OF_SCOPE:
        raise ValidationError(f"method {method!r} is not provided by the GPU LP engine "
                              f"(only {METHODS}); use the reference for MILP / A*")
    if method not in METHODS:
        raise ValidationError(f"unknown method {method!r} (one of {METHODS + OUT_OF_SCOPE})")
    if switch_mode == HYPER_EDGE:
        raise ValidationError("hyper-edge switches apply to the whole-chunk model only")
    notes: list[str] = []
    start = time.perf_counter()
    tau = epoch_duration(t, d.chunk_size, epoch_mode, em)
    opts = ModelOptions(switch_mode=switch_mode, buffer_limit=buffer_limit)
    cfg = EpochConfig(tau, 1, epoch_mode, em, d.chunk_size)
    if _benefits_from_copy(d):
        notes.append("demand is multicast: the copy-free program only bounds "
                     "what copy-capable schedules achieve")
        warnings.warn(notes[-1])
    sopts = SolverOptions(eps_rel=eps_rel, time_limit=time_limit, device=device)
    sol = None
    if epochs is None:
        epochs, sol = feasible_horizon(t, d, cfg, opts, device=device, sopts=sopts)
        notes.append(f"doubling search: horizon {epochs} is feasible")

    def builder(K: int):
        return build_from_plan(make_plan(t, d, cfg.with_horizon(K), opts), device)

    if search_horizon:
        if sol is not None:
            sol.model.close()
        k_star, sol = min_feasible_horizon(builder, 1, epochs, sopts)
    else:
        k_star = epochs
        if sol is None:
            sol = solve(builder(k_star), sopts)
    if not sol.feasible:
        if sol.status == INFEASIBLE:
            raise HorizonInfeasibleError(k_star, k_star)
        raise SolverTimeoutError(f"no solution within {time_limit}s")
    sched, x = schedule_with_flows(sol)  # x: the flows the events were peeled from
    if sched.meta:
        notes.append(f"loose solution polished to eps {sched.meta.get('polish_eps')} "
                     f"for an exact decomposition")
    check = check_lp_schedule(sol.model.plan, x, tol=check_tol, device=device)
    if not check.ok:
        raise ValidationError(f"refusing to emit schedule: flow replay found violations {check}")
    report = _checked_replay(sched, t, d, switch_mode)
    wall = time.perf_counter() - start
    return SynthesisResult(sched, report, method, sol.status, sol.solve_wall_time, wall,
                           sol.objective, sol.achieved_gap, k_star, tau, notes, check)


def _checked_replay(sched: Schedule, t: Topology, d: Demand, switch_mode: str) -> SimReport:
    """The reference's refuse-to-emit replay (workflow.py:125-132), on the
    native event simulator."""
    report = simulate(sched, t, d, SimOptions(switch_mode=switch_mode))
    if report.violations:
        kinds = sorted({v.kind for v in report.violations})
        raise ValidationError(
            f"refusing to emit schedule: replay found {len(report.violations)} "
            f"violations ({', '.join(kinds)})")
    return report


def _benefits_from_copy(d: Demand) -> bool:
    seen = set()
    for s, c, _ in d.entries:
        if (s, c) in seen:
            return True
        seen.add((s, c))
    return False
