"""Schedules from LP rates: per-chunk path events (reference lp.py:156-301).

The LP gives per-source link rates per epoch; a schedule says which fraction
of which chunk crosses which link in which epoch. Decomposition follows the
reference exactly -- reads are served earliest first, each read is traced
backwards through buffers (preferred) and arrivals (senders in str() order)
to the source's epoch-0 pool, the bottleneck is peeled off every arc -- so a
solution vector yields the same event list as collsched.lp_rates_to_schedule.
The reference re-sorts the whole flow dictionary at every hop (lp.py:257);
here each (node, arrival epoch) looks at its in-edges in a precomputed order.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .errors import ConservationError, SolverBackendError, ValidationError
from .lp import TOL, LpPlan, completion_of


@dataclass(frozen=True)
class ScheduleEvent:
    source: object
    chunk: int
    src: object
    dst: object
    epoch: int
    fraction: float = 1.0


@dataclass(frozen=True)
class Schedule:
    tau: float
    events: tuple
    completion_epoch: int
    chunk_size: int = 1
    meta: dict = field(default_factory=dict)

    @property
    def transfer_time(self) -> float:
        return (self.completion_epoch + 1) * self.tau if self.completion_epoch >= 0 else 0.0


def schedule_to_json(s: Schedule) -> dict:
    """Same document shape as the reference (schedule.py:217-229)."""
    return {"tau_sec": s.tau, "chunk_size_bytes": s.chunk_size,
            "completion_epoch": s.completion_epoch, "transfer_time_sec": s.transfer_time,
            "events": [{"src_rank": e.source, "chunk": e.chunk, "from": e.src, "to": e.dst,
                        "epoch": e.epoch, "fraction": e.fraction} for e in s.events],
            "meta": dict(s.meta)}


def save_schedule(s: Schedule, path) -> None:
    with open(path, "w") as f:
        json.dump(schedule_to_json(s), f, indent=2, sort_keys=True)
        f.write("\n")


def lp_rates_to_schedule(sol, t=None, d=None, cfg=None) -> Schedule:
    """Decompose an LP solution (from this package's solve) into fractional
    per-chunk events; raises ConservationError on residue, like the reference."""
    return schedule_with_flows(sol)[0]


def schedule_with_flows(sol) -> tuple:
    """(Schedule, x): the schedule and the exactly conserving flow vector its
    events were peeled from (the repaired / polished solution), for replay."""
    if not sol.feasible:
        raise ValidationError(f"cannot schedule a solution with status {sol.status}")
    plan: LpPlan = sol.model.plan
    meta = {}
    try:
        events, x = _decompose_solution(plan, sol.x)
    except ConservationError:
        # A loose first-order solution (e.g. eps_rel 1e-4) can leave a chunk
        # short by ~eps after the flow repair. Polish it on the device --
        # warm-started from this solution -- to POLISH_EPS and decompose that
        # (the reference's exact HiGHS solutions never need this).
        eps = sol.meta.get("eps_rel")
        if eps is None or eps <= POLISH_EPS or not hasattr(sol.model, "handle"):
            raise
        from .solver import SolverOptions, solve
        pol = solve(sol.model, SolverOptions(eps_rel=POLISH_EPS, device=sol.model.ctx.device,
                                             time_limit=600.0, max_iters=50_000_000), warm=sol)
        if not pol.feasible:
            raise
        meta = {"polished_from_eps": eps, "polish_eps": POLISH_EPS,
                "polish_iters": pol.meta["iters"], "polish_device_s": pol.meta["device_seconds"]}
        events, x = _decompose_solution(plan, pol.x)
        sol = pol
    # finish time of the flows the events were peeled from (the repaired /
    # polished x), the reference's lp_completion_epoch rule (lp.py:139-153)
    sched = Schedule(tau=plan.cfg.tau, events=tuple(events), completion_epoch=completion_of(plan, x),
                     chunk_size=plan.demand.chunk_size, meta=meta)
    return sched, x


POLISH_EPS = 1e-8


def _decompose_solution(plan: LpPlan, x) -> tuple:
    """(events, x'): the decomposition and the flow vector it was peeled from.

    1. A near-vertex solution (every pool's deficit <= RAW_OK, far below the
       reference's TOL) is decomposed exactly as the reference does it: the
       raw x with TOL = 1e-6 thresholds. For a unique optimum this gives the
       reference's event list (GPU solutions carry ~1e-9 noise, all below TOL).
    2. Otherwise (a looser first-order point) the flows are repaired to
       conserve exactly and peeled with the reference's TOL, then with DUST if
       TOL-sized remnants block a path.
    """
    x = np.asarray(x, dtype=np.float64)
    if max_deficit(plan, x) <= RAW_OK:
        try:
            return _native_or_residue(plan, x, TOL), x
        except ConservationError:
            pass
    xr = repair_flows(plan, x)
    # reads only shrink in the repair: a pair whose reads no longer add up to
    # its demand would end in a residue -- say so before peeling
    if plan.P and float((plan.pair_units - plan.rd_matrix(xr).sum(axis=1)).max()) > TOL:
        raise ConservationError("repaired flows deliver less than the demand")
    try:
        return _native_or_residue(plan, xr, TOL), xr
    except ConservationError:
        return _native_or_residue(plan, xr, DUST), xr


def _native_or_residue(plan: LpPlan, x: np.ndarray, tol: float) -> list:
    try:
        return decompose_native(plan, x, tol)
    except SolverBackendError as exc:  # the native decomposition reports residues as errors
        if "conservation residue" in str(exc) or "did not converge" in str(exc):
            raise ConservationError(str(exc)) from exc
        raise


RAW_OK = 1e-7  # pool deficits up to this: decompose x as is (reference procedure)
DUST = 1e-12  # peel threshold of last resort on repaired flows


def _pool_terms(plan: LpPlan, F, k, S, Nn, pair_of):
    """inflow(s,n) at epoch k, reads(s,n) at k, outflow(s,n) at epoch k+1."""
    K = plan.K
    inflow = np.zeros((S, Nn))
    kin = k - plan.delta
    ok = kin >= 0
    if ok.any():
        np.add.at(inflow, (slice(None), plan.edst[ok]), F[:, ok, kin[ok]])
    out = np.zeros((S, Nn))
    if k + 1 <= K - 1:
        np.add.at(out, (slice(None), plan.esrc), F[:, :, k + 1])
    return inflow, out


def _split(plan: LpPlan, x: np.ndarray):
    S, E, G, K = plan.S, plan.E, plan.G, plan.K
    F = np.stack([x[s * plan.SB:s * plan.SB + E * K].reshape(E, K) for s in range(S)]) if S else np.zeros((0, E, K))
    B = np.stack([x[s * plan.SB + E * K:(s + 1) * plan.SB].reshape(G, K + 1) for s in range(S)]) if S else np.zeros((0, G, K + 1))
    Rd = plan.rd_matrix(x).copy()
    gpu_nodes = np.flatnonzero(plan.is_switch == 0)
    pair_of = -np.ones((S, len(plan.nodes)), dtype=np.int64)
    pair_of[plan.pair_src, plan.pair_dst] = np.arange(plan.P)
    return F, B, Rd, gpu_nodes, pair_of


def max_deficit(plan: LpPlan, x: np.ndarray) -> float:
    """Largest amount any (source, node, epoch) pool sends or reads beyond
    what it holds plus what lands in it (0 for an exactly conserving flow)."""
    S, Nn, K = plan.S, len(plan.nodes), plan.K
    if S == 0:
        return 0.0
    F, B, Rd, gpu, pair_of = _split(plan, x)
    worst = 0.0
    hold = np.zeros((S, Nn))
    hold[:, gpu] = B[:, :, 0]
    for k in range(K):
        inflow, out = _pool_terms(plan, F, k, S, Nn, pair_of)
        reads = np.where(pair_of >= 0, Rd[np.maximum(pair_of, 0), k], 0.0)
        avail = hold + inflow
        worst = max(worst, float((reads + out - avail).max()))
        hold = np.zeros((S, Nn))
        hold[:, gpu] = B[:, :, k + 1]
    return worst


def repair_flows(plan: LpPlan, x: np.ndarray) -> np.ndarray:
    """Forward pass over epochs that scales down, at every pool whose
    next-epoch sends plus reads exceed what it holds plus its arrivals, those
    sends and reads to fit, and recomputes the buffers. Flows only shrink, so
    capacities still hold; reads shrink by the LP's residual (~eps_rel), so
    finish times are unchanged. Afterwards every read traces back to the
    source and decomposition cannot hit a dead end."""
    S, E, G, K, Nn = plan.S, plan.E, plan.G, plan.K, len(plan.nodes)
    if S == 0:
        return x
    F, B, Rd, gpu, pair_of = _split(plan, x)
    F = np.maximum(F, 0.0)
    Rd = np.maximum(Rd, 0.0)
    has_pair = pair_of >= 0
    pidx = np.maximum(pair_of, 0)
    # epoch-0 sends come out of the source's initial pool (init row, lp.py:69-72)
    out_units = np.zeros(S)
    np.add.at(out_units, plan.pair_src, plan.pair_units)
    s_idx = np.arange(S)
    out0 = np.zeros((S, Nn))
    np.add.at(out0, (slice(None), plan.esrc), F[:, :, 0])
    send0 = out0[s_idx, plan.snode]
    sc0 = np.where(send0 > out_units, out_units / np.maximum(send0, 1e-300), 1.0)
    src_is_s = plan.esrc[None, :] == plan.snode[:, None]
    F[:, :, 0] *= np.where(src_is_s, sc0[:, None], 1.0)
    hold = np.zeros((S, Nn))
    hold[s_idx, plan.snode] = np.maximum(out_units - send0 * sc0, 0.0)
    gpu_of = -np.ones(Nn, dtype=np.int64)
    gpu_of[gpu] = np.arange(len(gpu))
    B[:, :, 0] = hold[:, gpu]
    for k in range(K):
        inflow, out = _pool_terms(plan, F, k, S, Nn, pair_of)
        reads = np.where(has_pair, Rd[pidx, k], 0.0)
        avail = hold + inflow
        req = reads + out
        scale = np.where(req > avail, np.maximum(avail, 0.0) / np.maximum(req, 1e-300), 1.0)
        Rd[pidx[has_pair], k] = reads[has_pair] * scale[has_pair]
        if k + 1 <= K - 1:
            F[:, :, k + 1] *= scale[:, plan.esrc]
        nxt = np.maximum(avail - req * scale, 0.0)
        nxt[:, plan.is_switch.astype(bool)] = 0.0
        B[:, :, k + 1] = nxt[:, gpu]
        hold = nxt
    y = x.copy()
    for s in range(S):
        y[s * plan.SB:s * plan.SB + E * K] = F[s].reshape(-1)
        y[s * plan.SB + E * K:(s + 1) * plan.SB] = B[s].reshape(-1)
    base = S * plan.SB
    rr = y[base:base + plan.P * 2 * K].reshape(plan.P, K, 2)
    rr[:, :, 0] = Rd
    rr[:, :, 1] = np.cumsum(Rd, axis=1)
    return y


def _str_ranks(items) -> np.ndarray:
    """Position of every item in str() order (equal strings share a rank)."""
    keys = [str(v) for v in items]
    order = sorted(set(keys))
    pos = {k: i for i, k in enumerate(order)}
    return np.array([pos[k] for k in keys], dtype=np.int32)


def decompose_native(plan: LpPlan, x: np.ndarray, tol: float = TOL, need_tol: float = TOL,
                     threads: int = 0) -> list:
    """The decomposition in libteccl_b200 (csrc/schedule.cu, one CPU thread per
    source); same events as decompose() below."""
    import ctypes as C
    from . import _native as nat
    lib = nat.load()
    nodes, E = plan.nodes, plan.E
    order_in = sorted(range(E), key=lambda e: (int(plan.edst[e]), str(nodes[int(plan.esrc[e])])))
    in_edges = np.array(order_in, dtype=np.int32)
    in_ptr = np.zeros(len(nodes) + 1, dtype=np.int32)
    np.add.at(in_ptr, plan.edst.astype(np.int64) + 1, 1)
    in_ptr = np.cumsum(in_ptr).astype(np.int32)
    by_pair: dict = {}
    for s, c, dst in sorted(plan.demand.entries, key=lambda e: (str(e[0]), e[1], str(e[2]))):
        by_pair.setdefault((s, dst), []).append(c)
    pair_index = {pair: p for p, (pair, _) in enumerate(plan.pairs)}
    chunks = [by_pair.get(pair, []) for pair, _ in plan.pairs]
    pcp = np.zeros(plan.P + 1, dtype=np.int32)
    pcp[1:] = np.cumsum([len(c) for c in chunks])
    pch = np.array([c for cs in chunks for c in cs], dtype=np.int32)
    porder = np.array([pair_index[pair] for pair, _ in sorted(by_pair.items(), key=str)],
                      dtype=np.int32)
    srank = _str_ranks(plan.sources)
    nrank = _str_ranks(nodes)
    x = np.ascontiguousarray(x, dtype=np.float64)
    h = C.c_void_p()
    cnt = C.c_int64()
    nat.check(lib.teccl_schedule_te(
        C.byref(plan.desc()), nat.ptr(x, C.c_double), float(tol), float(need_tol),
        nat.ptr(in_ptr, C.c_int32), nat.ptr(in_edges, C.c_int32), nat.ptr(pcp, C.c_int32),
        nat.ptr(pch if pch.size else np.zeros(1, np.int32), C.c_int32),
        nat.ptr(porder if porder.size else np.zeros(1, np.int32), C.c_int32),
        nat.ptr(srank if srank.size else np.zeros(1, np.int32), C.c_int32),
        nat.ptr(nrank, C.c_int32), int(threads), C.byref(h), C.byref(cnt)))
    n = cnt.value
    ss, cc, ee, kk = (np.empty(max(n, 1), np.int32) for _ in range(4))
    ff = np.empty(max(n, 1), np.float64)
    nat.check(lib.teccl_schedule_fetch(h, nat.ptr(ss, C.c_int32), nat.ptr(cc, C.c_int32),
                                       nat.ptr(ee, C.c_int32), nat.ptr(kk, C.c_int32),
                                       nat.ptr(ff, C.c_double)))
    if n == 0:
        return []
    node_arr = np.empty(len(nodes), dtype=object)
    node_arr[:] = list(nodes)
    src_arr = np.empty(len(plan.sources), dtype=object)
    src_arr[:] = list(plan.sources)
    e = ee[:n]
    return list(map(ScheduleEvent, src_arr[ss[:n]].tolist(), cc[:n].tolist(),
                    node_arr[plan.esrc[e]].tolist(), node_arr[plan.edst[e]].tolist(),
                    kk[:n].tolist(), ff[:n].tolist()))


def decompose(plan: LpPlan, x: np.ndarray, tol: float = TOL, need_tol: float = TOL) -> list:
    """Readable restatement of the reference's decomposition (lp.py:156-301),
    kept as the specification the native version is tested against. tol:
    entries at or below it count as empty while tracing (the reference's 1e-6);
    need_tol: unserved remainder accepted per chunk."""
    K, E = plan.K, plan.E
    nodes = plan.nodes
    esrc, edst, delta = plan.esrc, plan.edst, plan.delta
    gpu_of = {}
    g = 0
    for i, n in enumerate(nodes):
        if not plan.is_switch[i]:
            gpu_of[i] = g
            g += 1
    # in-edges of every node, in the order the reference scans them: by
    # str(sender) (lp.py:257 sorts keys by (str(dst), str(src), epoch))
    in_edges = {i: [] for i in range(len(nodes))}
    for e in range(E):
        in_edges[int(edst[e])].append(e)
    for i in in_edges:
        in_edges[i].sort(key=lambda e: str(nodes[int(esrc[e])]))
    # demanded chunk ids per (source, destination), in the reference order
    by_pair: dict = {}
    for s, c, dst in sorted(plan.demand.entries, key=lambda e: (str(e[0]), e[1], str(e[2]))):
        by_pair.setdefault((s, dst), []).append(c)
    pair_index = {pair: p for p, (pair, _) in enumerate(plan.pairs)}
    node_index = {n: i for i, n in enumerate(nodes)}
    esrc = [int(v) for v in esrc]
    edst = [int(v) for v in edst]
    delta = [int(v) for v in delta]
    events = []
    for si, s in enumerate(plan.sources):
        b = si * plan.SB
        fres = x[b:b + E * K].reshape(E, K).tolist()
        bres = x[b + E * K:b + plan.SB].reshape(plan.G, K + 1).tolist()
        snode = int(plan.snode[si])
        for (s2, dst), chunk_ids in sorted(by_pair.items(), key=str):
            if s2 != s:
                continue
            p = pair_index[(s, dst)]
            rres = plan.rd_matrix(x)[p].tolist()
            dn = node_index[dst]
            cursor = 0  # reads only shrink: the earliest live read never moves back
            for c in chunk_ids:
                need = 1.0
                guard = 0
                while need > need_tol:
                    guard += 1
                    if guard > 10000:
                        raise ConservationError("path peeling did not converge")
                    while cursor < K and not rres[cursor] > tol:
                        cursor += 1
                    if cursor >= K:
                        raise ConservationError(
                            f"conservation residue: chunk {c} of {s!r} short by {need:.2e} at {dst!r}")
                    k_read = cursor
                    got, path = _peel(snode, dn, k_read, min(need, rres[k_read]), fres, bres,
                                      in_edges, esrc, delta, gpu_of, tol)
                    if got <= tol:
                        raise ConservationError(
                            f"conservation residue: no backing path for read at epoch {k_read}")
                    rres[k_read] -= got
                    if rres[k_read] <= tol:
                        rres[k_read] = 0.0
                    need -= got
                    for (e, tt, frac) in path:
                        events.append(ScheduleEvent(s, c, nodes[esrc[e]], nodes[edst[e]],
                                                    tt, frac))
            # the reference keeps one rres dict per source across its pairs;
            # pairs of one source have distinct destinations, so per-pair
            # copies are equivalent
    events.sort(key=lambda e: (e.epoch, str(e.source), str(e.src), str(e.dst), e.chunk))
    merged: dict = {}
    for e in events:
        key = (e.source, e.chunk, e.src, e.dst, e.epoch)
        merged[key] = merged.get(key, 0.0) + e.fraction
    return [ScheduleEvent(s, c, i, j, k, f) for (s, c, i, j, k), f in sorted(
        merged.items(), key=lambda kv: (kv[0][4], str(kv[0][0]), str(kv[0][2]), str(kv[0][3]),
                                        kv[0][1]))]


def _peel(snode, dst, k_read, amount, fres, bres, in_edges, esrc, delta, gpu_of, tol):
    """One backward path from a read to the source's epoch-0 pool
    (reference lp.py:235-291); returns (fraction, [(edge, send_epoch, fraction)])."""
    arcs = []
    node, k = dst, k_read
    while True:
        if node == snode and k == 0:
            break
        g = gpu_of.get(node)
        carry = bres[g][k] if g is not None else 0.0
        if carry > tol:
            arcs.append((0, g, k))
            k -= 1
            if k < 0:
                raise ConservationError("buffer traces past epoch 0")
            continue
        found = None
        for e in in_edges[node]:
            tt = k - delta[e]
            if tt >= 0 and fres[e][tt] > tol:
                found = (e, tt)
                break
        if found is None:
            return 0.0, []
        arcs.append((1, found[0], found[1]))
        e, tt = found
        if tt == 0:
            if esrc[e] != snode:
                return 0.0, []
            break
        node, k = esrc[e], tt - 1
    bottleneck = amount
    for kind, a, bb in arcs:
        bottleneck = min(bottleneck, bres[a][bb] if kind == 0 else fres[a][bb])
    if bottleneck <= tol:
        return 0.0, []
    out = []
    for kind, a, bb in arcs:
        row = bres[a] if kind == 0 else fres[a]
        row[bb] -= bottleneck
        if row[bb] <= tol:
            row[bb] = 0.0
        if kind == 1:
            out.append((a, bb, bottleneck))
    return bottleneck, out
