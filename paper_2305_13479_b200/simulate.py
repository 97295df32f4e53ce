"""Event-level replay of a schedule (reference simulator.py:25-266).

Same types and entry points as collsched.simulator -- SimOptions, Violation,
SimReport, simulate(sched, t, d, opts), algorithmic_bandwidth -- with the
replay itself in libteccl_b200.so (csrc/simulate.cu, teccl_simulate): the
schedule's event list is replayed event by event for causality (a send needs
data the sender holds), per-(edge, window) capacity, switch arrivals resting
past their forwarding epoch and unmet demand. This module only does what is
O(edges + entries): the exact rational per-edge arithmetic
(simulator.py:76-92), input validation (:96-102) and the formatting and
ordering of the violations (:165-189). The hyper-edge switch mode belongs to
the whole-chunk MILP path (out of scope) and is rejected.
"""

from __future__ import annotations

import ctypes as C
from collections import Counter
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _native as nat
from .demand import check_demand_nodes
from .epochs import ceil_q, snap
from .errors import ScheduleError, ValidationError
from .lp import COPY, HYPER_EDGE, NO_COPY
from .topology import require_valid

WHOLE = 1.0 - 1e-9  # simulator.py:22


@dataclass(frozen=True)
class SimOptions:
    switch_mode: str = COPY
    tolerance: float = 1e-6

    def __post_init__(self):
        if self.switch_mode not in (COPY, NO_COPY, HYPER_EDGE):
            raise ValidationError(f"unknown switch mode {self.switch_mode!r}")


@dataclass(frozen=True)
class Violation:
    kind: str  # capacity | causality | switch-buffer | unmet-demand
    location: str
    epoch: int


@dataclass
class SimReport:
    violations: list
    completion_epochs: dict  # destination -> last demanded arrival epoch
    completion_epoch: int
    transfer_time: float
    output_buffer_bytes: dict
    demand_bytes: int
    tau: float
    per_entry_completion: dict = field(default_factory=dict)

    @property
    def ok(self) -> bool:
        return not self.violations


def _str_ranks(items) -> np.ndarray:
    keys = [str(v) for v in items]
    pos = {k: i for i, k in enumerate(sorted(set(keys)))}
    return np.array([pos[k] for k in keys], dtype=np.int32)


def simulate(sched, t, d, opts: SimOptions | None = None, threads: int = 0) -> SimReport:
    """Replay `sched` against topology `t` and demand `d` (simulator.py:58-208)."""
    opts = opts or SimOptions()
    require_valid(t)
    check_demand_nodes(d, t)
    if opts.switch_mode == HYPER_EDGE:
        raise ValidationError("hyper-edge replay belongs to the whole-chunk path; "
                              "the LP engine emits copy / no-copy schedules")
    tol = opts.tolerance
    tau = snap(sched.tau)
    if tau <= 0:
        raise ScheduleError("schedule has non-positive epoch duration")
    chunk = Fraction(sched.chunk_size)
    nodes = list(t.nodes)
    nidx = {n: i for i, n in enumerate(nodes)}
    edges = list(t.edges)
    eidx = {(e.src, e.dst): i for i, e in enumerate(edges)}
    caps = [snap(e.capacity) * tau / chunk for e in edges]

    events = sched.events
    n = len(events)
    frac = np.fromiter((ev.fraction for ev in events), dtype=np.float64, count=n)
    epoch = np.fromiter((ev.epoch for ev in events), dtype=np.int64, count=n)
    edge = np.fromiter((eidx.get((ev.src, ev.dst), -1) for ev in events), dtype=np.int64, count=n)
    bad = (edge < 0) | (epoch < 0) | ~((frac > 0.0) & (frac <= 1.0 + tol))
    if bad.any():  # the first offender in replay order raises (simulator.py:96-102)
        ev = min((events[i] for i in np.flatnonzero(bad)),
                 key=lambda e: (e.epoch, str(e.source), str(e.src), str(e.dst), e.chunk))
        if (ev.src, ev.dst) not in eidx:
            raise ScheduleError(f"event references unknown edge ({ev.src!r},{ev.dst!r})")
        if ev.epoch < 0:
            raise ScheduleError(f"event at negative epoch {ev.epoch}")
        raise ScheduleError(f"event fraction {ev.fraction} outside (0, 1]")

    whole_only = bool((frac >= WHOLE).all())
    kap = [max(1, ceil_q(1 / c)) if whole_only else 1 for c in caps]
    widen = max(kap, default=1) - 1
    delta = np.array([ceil_q(snap(e.alpha) / tau) + widen for e in edges], dtype=np.int32)
    window = np.array(kap, dtype=np.int32)
    budget = np.array([float(w * c) for w, c in zip(kap, caps)], dtype=np.float64)
    is_sw = np.array([1 if t.is_switch(v) else 0 for v in nodes], dtype=np.uint8)

    entries = list(d.entries)
    ent_s = np.array([nidx[s] for s, _, _ in entries], dtype=np.int32)
    ent_c = np.array([c for _, c, _ in entries], dtype=np.int32)
    ent_d = np.array([nidx[x] for _, _, x in entries], dtype=np.int32)
    try:
        ev_s = np.fromiter((nidx[ev.source] for ev in events), dtype=np.int32, count=n)
    except KeyError as exc:  # (the reference would report every such send as causality)
        raise ScheduleError(f"event names source {exc.args[0]!r}, which is not a node") from None
    ev_c = np.fromiter((ev.chunk for ev in events), dtype=np.int32, count=n)
    e32 = edge.astype(np.int32)
    ev_src = np.array([nidx[e.src] for e in edges], dtype=np.int32)[e32] if n else np.zeros(0, np.int32)
    ev_dst = np.array([nidx[e.dst] for e in edges], dtype=np.int32)[e32] if n else np.zeros(0, np.int32)
    k32 = epoch.astype(np.int32)
    nrank = _str_ranks(nodes)

    desc = nat.SimDesc()
    desc.num_nodes = len(nodes)
    desc.node_is_switch = nat.ptr(is_sw, C.c_uint8)
    desc.num_edges = len(edges)
    desc.edge_delta = nat.ptr(delta, C.c_int32)
    desc.edge_window = nat.ptr(window, C.c_int32)
    desc.edge_budget = nat.ptr(budget, C.c_double)
    desc.num_entries = len(entries)
    z = np.zeros(1, np.int32)
    desc.entry_source = nat.ptr(ent_s if len(entries) else z, C.c_int32)
    desc.entry_chunk = nat.ptr(ent_c if len(entries) else z, C.c_int32)
    desc.entry_dst = nat.ptr(ent_d if len(entries) else z, C.c_int32)
    desc.switch_mode = 1 if opts.switch_mode == NO_COPY else 0
    desc.tolerance = float(tol)

    lib = nat.load()
    h = C.c_void_p()
    counts = np.zeros(4, np.int64)
    zf = np.zeros(1, np.float64)
    arg = lambda a, ct, fb=z: nat.ptr(a if a.size else fb, ct)  # noqa: E731
    nat.check(lib.teccl_simulate(
        C.byref(desc), n, arg(ev_s, C.c_int32), arg(ev_c, C.c_int32), arg(ev_src, C.c_int32),
        arg(ev_dst, C.c_int32), arg(e32, C.c_int32), arg(k32, C.c_int32), arg(frac, C.c_double, zf),
        nat.ptr(nrank, C.c_int32), nat.ptr(nrank, C.c_int32), int(threads), C.byref(h),
        nat.ptr(counts, C.c_int64)))
    n0, n1, n2, n3 = (int(v) for v in counts)
    caus = np.empty(max(n0, 1), np.int64)
    capv = np.empty(max(2 * n1, 1), np.int64)
    swv = np.empty(max(4 * n2, 1), np.int64)
    done = np.empty(max(n3, 1), np.int32)
    nat.check(lib.teccl_simulate_fetch(h, nat.ptr(caus, C.c_int64), nat.ptr(capv, C.c_int64),
                                       nat.ptr(swv, C.c_int64), nat.ptr(done, C.c_int32)))

    violations = []
    for i in caus[:n0]:
        ev = events[int(i)]
        violations.append(Violation("causality", f"{ev.src!r} lacks chunk "
                                    f"{ev.chunk} of {ev.source!r}", ev.epoch))
    for q in range(n1):
        e = edges[int(capv[2 * q])]
        violations.append(Violation("capacity", f"({e.src!r},{e.dst!r})", int(capv[2 * q + 1])))
    rest = [(nodes[int(swv[4 * q])], int(swv[4 * q + 1]), nodes[int(swv[4 * q + 2])],
             int(swv[4 * q + 3])) for q in range(n2)]
    rest.sort(key=lambda r: str((r[0], r[1], r[2])))  # stable: records keep their order
    for s, c, sw, usable in rest:
        violations.append(Violation("switch-buffer", f"chunk {c} of {s!r} rests at {sw!r}", usable))

    done_of = {ent: int(done[i]) for i, ent in enumerate(entries)}
    per_entry: dict = {}
    for ent in sorted(done_of, key=str):
        k = done_of[ent]
        if k < 0:
            s, c, dst = ent
            violations.append(Violation("unmet-demand", f"chunk {c} of {s!r} at {dst!r}", -1))
        else:
            per_entry[ent] = k
    completion_per_dest: dict = {}
    for (s, c, dst), k in per_entry.items():
        completion_per_dest[dst] = max(completion_per_dest.get(dst, -1), k)
    completion = max(per_entry.values(), default=-1)
    received = Counter(dst for (_, _, dst) in entries)
    output_bytes = {v: d.chunk_size * received[v] for v in nodes if not t.is_switch(v)}
    return SimReport(
        violations=violations, completion_epochs=completion_per_dest, completion_epoch=completion,
        transfer_time=(completion + 1) * float(tau) if completion >= 0 else 0.0,
        output_buffer_bytes=output_bytes, demand_bytes=d.total_bytes(), tau=float(tau),
        per_entry_completion=per_entry)


def algorithmic_bandwidth(report: SimReport) -> dict:
    """Received bytes over transfer time, per destination and in aggregate
    (simulator.py:258-266)."""
    total = sum(report.output_buffer_bytes.values())
    if total == 0:
        return {"aggregate": 0.0, "per_node": {v: 0.0 for v in report.output_buffer_bytes}}
    if report.transfer_time <= 0:
        raise ValidationError("zero transfer time with nonzero demand")
    per_node = {v: b / report.transfer_time for v, b in report.output_buffer_bytes.items()}
    return {"aggregate": total / report.transfer_time, "per_node": per_node}
