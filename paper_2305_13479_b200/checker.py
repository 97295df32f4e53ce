"""(4) Exact-integer schedule checker / epoch simulator on the GPU.

Replays an LP solution of the time-expanded model in fixed-point integer
units (`quantum` units per chunk): capacity per (edge, epoch), buffer
causality per (source, node, epoch), switch pass-through, and per-pair
demand satisfaction, plus the completion epoch. Replaces the reference's
simulate() (pkg/src/collsched/simulator.py:58-235) at the flow level for LP
solutions; the event list itself is replayed by simulate.py.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .lp import LpPlan

DEFAULT_QUANTUM = 1 << 30


@dataclass(frozen=True)
class CheckReport:
    capacity_violations: int
    causality_violations: int
    switch_violations: int
    unmet_pairs: int
    completion_epoch: int
    max_capacity_excess: float   # chunks
    max_buffer_deficit: float    # chunks

    @property
    def ok(self) -> bool:
        return not (self.capacity_violations or self.causality_violations or
                    self.switch_violations or self.unmet_pairs)


def check_lp_schedule(plan: LpPlan, x: np.ndarray, tol: float = 1e-6,
                      quantum: int = DEFAULT_QUANTUM, device: int = 0) -> CheckReport:
    """tol is the per-check slack in chunks (reference simulator tolerance)."""
    ctx = nat.Context.get(device)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape[0] != plan.num_vars:
        raise ValueError(f"solution has {x.shape[0]} entries, plan expects {plan.num_vars}")
    rep = nat.CheckReport()
    slack = int(np.ceil(tol * quantum))
    nat.check(ctx.lib.teccl_check_te(ctx.handle, C.byref(plan.desc()), nat.ptr(x, C.c_double),
                                     int(quantum), slack, C.byref(rep)))
    return CheckReport(int(rep.capacity_violations), int(rep.causality_violations),
                       int(rep.switch_violations), int(rep.unmet_pairs),
                       int(rep.completion_epoch), rep.max_capacity_excess / quantum,
                       rep.max_buffer_deficit / quantum)
