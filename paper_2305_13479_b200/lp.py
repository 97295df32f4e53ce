"""Copy-free time-expanded LP: host plan + device-built model.

Drop-in for the reference's `build_lp_model` / `lp_completion_epoch`
(pkg/src/collsched/lp.py:22-153). The host computes only the compact
tables (node kinds, edges with delay and per-epoch capacity, sorted sources,
sorted demand pairs) using the reference's exact ordering and rational
arithmetic; the CUDA builder (csrc/te_build.cu) expands them into CSR/CSC
directly in HBM. Variable and row order equal the reference's, so a solution
vector from either side indexes the same variables.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .demand import check_demand_nodes
from .epochs import EpochConfig, cap_chunks, compute_delta
from .errors import ConservationError, ValidationError
from .topology import require_valid

COPY = "copy"
NO_COPY = "no-copy"
HYPER_EDGE = "hyper-edge"
TOL = 1e-6  # reference lp.py:19


@dataclass(frozen=True)
class ModelOptions:
    """Same fields and checks as the reference (milp.py:159-171)."""
    switch_mode: str = COPY
    buffer_limit: float | None = None
    capacity_mode: str = "auto"

    def __post_init__(self):
        if self.switch_mode not in (COPY, NO_COPY, HYPER_EDGE):
            raise ValidationError(f"unknown switch mode {self.switch_mode!r}")
        if self.capacity_mode not in ("auto", "plain", "windowed"):
            raise ValidationError(f"unknown capacity mode {self.capacity_mode!r}")
        if self.buffer_limit is not None and self.buffer_limit <= 0:
            raise ValidationError("buffer_limit must be positive")


@dataclass
class LpPlan:
    """Compact description of one time-expanded LP (reference order)."""
    topology: object
    demand: object
    cfg: EpochConfig
    opts: ModelOptions
    nodes: list
    is_switch: np.ndarray      # uint8 [Nn]
    esrc: np.ndarray           # int32 [E]
    edst: np.ndarray           # int32 [E]
    delta: np.ndarray          # int32 [E]
    cap: np.ndarray            # float64 [E*K]
    sources: list
    snode: np.ndarray          # int32 [S]
    pairs: list                # [((s, dst), units)] sorted like lp.py:60
    pair_src: np.ndarray       # int32 [P] source slot
    pair_dst: np.ndarray       # int32 [P] node index
    pair_units: np.ndarray     # float64 [P]
    K: int
    buffer_limit: float
    phase1: bool = False          # feasibility LP (see feasibility_gap)
    _desc: object = field(default=None, repr=False)

    @property
    def E(self) -> int:
        return len(self.esrc)

    @property
    def S(self) -> int:
        return len(self.sources)

    @property
    def P(self) -> int:
        return len(self.pairs)

    @property
    def G(self) -> int:
        return int(len(self.nodes) - self.is_switch.sum())

    @property
    def SB(self) -> int:
        return self.E * self.K + self.G * (self.K + 1)

    @property
    def num_vars(self) -> int:
        return self.S * self.SB + self.P * 2 * self.K

    @property
    def num_rows(self) -> int:
        K, Nn, G = self.K, len(self.nodes), self.G
        rows = self.S + self.E * K + self.S * (Nn * K + G - 1) + self.P * K
        if self.buffer_limit >= 0:
            rows += G * (K + 1)
        return rows

    # variable indices (csrc/te_build.cu layout, = reference lp.py:47-65 order)
    def var_F(self, s: int, e: int, k: int) -> int:
        return s * self.SB + e * self.K + k

    def var_B(self, s: int, g: int, k: int) -> int:
        return s * self.SB + self.E * self.K + g * (self.K + 1) + k

    def var_Rd(self, p: int, k: int) -> int:
        return self.S * self.SB + p * 2 * self.K + 2 * k

    def var_Rc(self, p: int, k: int) -> int:
        return self.var_Rd(p, k) + 1

    def rc_matrix(self, x: np.ndarray) -> np.ndarray:
        """Cumulative reads Rc as a [P, K] view of a solution vector."""
        base = self.S * self.SB
        return x[base:base + self.P * 2 * self.K].reshape(self.P, self.K, 2)[:, :, 1]

    def rd_matrix(self, x: np.ndarray) -> np.ndarray:
        base = self.S * self.SB
        return x[base:base + self.P * 2 * self.K].reshape(self.P, self.K, 2)[:, :, 0]

    def flow_tensor(self, x: np.ndarray) -> np.ndarray:
        """F as [S, E, K]."""
        out = np.empty((self.S, self.E, self.K))
        for s in range(self.S):
            b = s * self.SB
            out[s] = x[b:b + self.E * self.K].reshape(self.E, self.K)
        return out

    def desc(self) -> nat.TeDesc:
        """C descriptor over this plan's arrays (kept alive by the plan)."""
        if self._desc is None:
            d = nat.TeDesc()
            d.num_nodes = len(self.nodes)
            d.num_edges = self.E
            d.num_sources = self.S
            d.num_pairs = self.P
            d.K = self.K
            d.node_is_switch = nat.ptr(self.is_switch, C.c_uint8)
            d.edge_src = nat.ptr(self.esrc, C.c_int32)
            d.edge_dst = nat.ptr(self.edst, C.c_int32)
            d.edge_delta = nat.ptr(self.delta, C.c_int32)
            d.edge_cap = nat.ptr(self.cap, C.c_double)
            d.source_node = nat.ptr(self.snode, C.c_int32)
            d.pair_source = nat.ptr(self.pair_src, C.c_int32)
            d.pair_dst = nat.ptr(self.pair_dst, C.c_int32)
            d.pair_units = nat.ptr(self.pair_units, C.c_double)
            d.buffer_limit = float(self.buffer_limit)
            d.phase1 = 1 if self.phase1 else 0
            self._desc = d
        return self._desc


def make_plan(t, d, cfg: EpochConfig, opts: ModelOptions | None = None) -> LpPlan:
    """Host tables in the reference's order (lp.py:27-45, 60, 74-77)."""
    opts = opts or ModelOptions()
    require_valid(t)
    check_demand_nodes(d, t)
    K = cfg.K
    nodes = list(t.nodes)
    nidx = {n: i for i, n in enumerate(nodes)}
    is_switch = np.array([1 if t.is_switch(n) else 0 for n in nodes], dtype=np.uint8)
    edges = list(t.edges)
    esrc = np.array([nidx[e.src] for e in edges], dtype=np.int32)
    edst = np.array([nidx[e.dst] for e in edges], dtype=np.int32)
    delta = np.array([compute_delta(e, cfg.tau) for e in edges], dtype=np.int32)
    cap = np.empty(len(edges) * K, dtype=np.float64)
    overrides = getattr(t, "capacity_overrides", {}) or {}
    over_edges = {(s, dd) for (s, dd, _k) in overrides}
    for i, e in enumerate(edges):
        if (e.src, e.dst) in over_edges:
            cap[i * K:(i + 1) * K] = [float(cap_chunks(t, e, k, cfg)) for k in range(K)]
        else:
            cap[i * K:(i + 1) * K] = float(cap_chunks(t, e, 0, cfg))
    sources = sorted({s for s, _, _ in d.entries}, key=str)
    sidx = {s: i for i, s in enumerate(sources)}
    units: dict = {}
    for s, _, dst in d.entries:
        units[(s, dst)] = units.get((s, dst), 0) + 1
    pairs = sorted(units.items(), key=str)
    return LpPlan(
        topology=t, demand=d, cfg=cfg, opts=opts, nodes=nodes, is_switch=is_switch,
        esrc=esrc, edst=edst, delta=delta, cap=cap, sources=sources,
        snode=np.array([nidx[s] for s in sources], dtype=np.int32), pairs=pairs,
        pair_src=np.array([sidx[s] for (s, _), _ in pairs], dtype=np.int32),
        pair_dst=np.array([nidx[dst] for (_, dst), _ in pairs], dtype=np.int32),
        pair_units=np.array([float(u) for _, u in pairs], dtype=np.float64),
        K=K, buffer_limit=float(opts.buffer_limit) if opts.buffer_limit is not None else -1.0)


class DeviceLP:
    """An LP resident in HBM (CSR + CSC + bounds + costs). `plan` is set for
    time-expanded models built by build_lp_model, None for generic uploads."""

    def __init__(self, handle, ctx: nat.Context, plan: LpPlan | None, name: str = "lp"):
        self.handle = handle
        self.ctx = ctx
        self.plan = plan
        self.name = name
        m, n, nnz = C.c_int32(), C.c_int32(), C.c_int64()
        nat.check(ctx.lib.teccl_lp_dims(handle, C.byref(m), C.byref(n), C.byref(nnz)))
        self.num_rows, self.num_vars, self.nnz = m.value, n.value, nnz.value
        self.meta: dict = {}
        if plan is not None:
            self.meta.update({
                "kind": "lp", "topology": plan.topology, "eff_topology": plan.topology,
                "demand": plan.demand, "cfg": plan.cfg, "opts": plan.opts,
                "delta": {(e.src, e.dst): int(dl) for e, dl in zip(plan.topology.edges, plan.delta)},
                "units": dict(plan.pairs), "sources": plan.sources, "windowed": False,
            })

    def export(self) -> dict:
        """Copy the model back to the host as canonical CSR arrays."""
        m, n, nnz = self.num_rows, self.num_vars, self.nnz
        out = {"row_ptr": np.empty(m + 1, np.int64), "col": np.empty(nnz, np.int32),
               "val": np.empty(nnz, np.float64), "row_lo": np.empty(m), "row_hi": np.empty(m),
               "var_lb": np.empty(n), "var_ub": np.empty(n), "obj": np.empty(n)}
        nat.check(self.ctx.lib.teccl_lp_export(
            self.handle, nat.ptr(out["row_ptr"], C.c_int64), nat.ptr(out["col"], C.c_int32),
            nat.ptr(out["val"], C.c_double), nat.ptr(out["row_lo"], C.c_double),
            nat.ptr(out["row_hi"], C.c_double), nat.ptr(out["var_lb"], C.c_double),
            nat.ptr(out["var_ub"], C.c_double), nat.ptr(out["obj"], C.c_double)))
        return out

    def export_csc(self) -> dict:
        n, nnz = self.num_vars, self.nnz
        out = {"col_ptr": np.empty(n + 1, np.int64), "row": np.empty(nnz, np.int32),
               "val": np.empty(nnz, np.float64)}
        nat.check(self.ctx.lib.teccl_lp_export_csc(
            self.handle, nat.ptr(out["col_ptr"], C.c_int64), nat.ptr(out["row"], C.c_int32),
            nat.ptr(out["val"], C.c_double)))
        return out

    def spmv_bench(self, reps: int = 50) -> tuple[float, float]:
        ms, by = C.c_double(), C.c_double()
        nat.check(self.ctx.lib.teccl_spmv_bench(self.ctx.handle, self.handle, int(reps),
                                                 C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def apply(self, v: np.ndarray, transpose: bool = False, matrix_free: int = 1) -> dict:
        """A.v (or A^T.v) on the device with the bounds (and costs) that path
        sees: matrix_free = 0 stored CSR/CSC, 1 per-entry matrix-free
        operator, 2 segment walkers (the PDLP kernels' operator)."""
        nin, nout = (self.num_rows, self.num_vars) if transpose else (self.num_vars, self.num_rows)
        return apply_operator(self.ctx, self.handle, v, nin, nout, transpose, matrix_free)

    def step_bench(self, reps: int = 50, pdlp: dict | None = None) -> dict:
        """Per-launch device time and algorithmic bytes of the fused kernels;
        `pdlp` overrides teccl_pdlp_opts fields (e.g. {"matrix_free": 2})."""
        return step_bench(self.ctx, self.handle, reps, pdlp)

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.teccl_lp_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def apply_operator(ctx, handle, v: np.ndarray, nin: int, nout: int, transpose: bool,
                   matrix_free: int) -> dict:
    """teccl_lp_apply: A.v / A^T.v with the bounds (and costs) of the chosen
    operator; `v` spans the gather window (the whole vector on one device)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (nin,):
        raise ValueError(f"expected a vector of length {nin}")
    out = {k: np.empty(nout, np.float64) for k in ("y", "lo", "hi")}
    out["cost"] = np.empty(nout if transpose else 1, np.float64)
    nat.check(ctx.lib.teccl_lp_apply(
        ctx.handle, handle, int(bool(transpose)), int(matrix_free),
        nat.ptr(v, C.c_double), nat.ptr(out["y"], C.c_double), nat.ptr(out["lo"], C.c_double),
        nat.ptr(out["hi"], C.c_double), nat.ptr(out["cost"], C.c_double)))
    if not transpose:
        del out["cost"]
    return out


def step_bench(ctx, handle, reps: int = 50, pdlp: dict | None = None) -> dict:
    """teccl_pdlp_step_bench[_opts]: per-launch time (CUDA events) and
    algorithmic bytes of the two half-step kernels after the real setup."""
    out = (C.c_double * 6)()
    if pdlp:
        o = nat.PdlpOpts()
        ctx.lib.teccl_pdlp_default_opts(C.byref(o))
        for k, v in pdlp.items():
            setattr(o, k, type(getattr(o, k))(v))
        nat.check(ctx.lib.teccl_pdlp_step_bench_opts(ctx.handle, handle, C.byref(o), int(reps), out))
    else:
        nat.check(ctx.lib.teccl_pdlp_step_bench(ctx.handle, handle, int(reps), out))
    return {"ms_col": out[0], "ms_row": out[1], "bytes_col": out[2], "bytes_row": out[3],
            "dict": out[4] == 1.0, "matrix_free": int(out[4]) if out[4] >= 2.0 else 0,
            "slice": int(out[5])}


def build_lp_model(t, d, cfg: EpochConfig, opts: ModelOptions | None = None,
                   device: int = 0, slot: int = 0) -> DeviceLP:
    """Build the copy-free TE-CCL LP on the GPU (reference lp.py:22-136);
    `slot` selects the device's context / stream (concurrent solves)."""
    plan = make_plan(t, d, cfg, opts)
    return build_from_plan(plan, device, slot)


def build_from_plan(plan: LpPlan, device: int = 0, slot: int = 0) -> DeviceLP:
    ctx = nat.Context.get(device, slot)
    h = C.c_void_p()
    nat.check(ctx.lib.teccl_lp_build_te(ctx.handle, C.byref(plan.desc()), C.byref(h)))
    return DeviceLP(h, ctx, plan, name="lp-alltoall")


def lp_completion_epoch(sol, tol: float = TOL) -> int:
    """Earliest epoch by which every pair's cumulative reads meet its demand
    (reference lp.py:139-153), vectorised over pairs."""
    return completion_of(sol.model.plan, sol.x, tol)


def completion_of(plan: "LpPlan", x, tol: float = TOL) -> int:
    """lp_completion_epoch of a solution vector x of `plan`'s LP."""
    rc = plan.rc_matrix(x)
    need = plan.pair_units - tol * np.maximum(1.0, plan.pair_units)
    ok = rc >= need[:, None]
    if not ok.any(axis=1).all():
        bad = int(np.argmin(ok.any(axis=1)))
        s, dst = plan.pairs[bad][0]
        raise ConservationError(f"pair ({s!r},{dst!r}) never reaches its demand")
    return int(ok.argmax(axis=1).max()) if plan.P else 0


def feasibility_gap(plan: LpPlan, device: int = 0, eps_rel: float = 1e-7,
                    max_iters: int = 2_000_000, time_limit: float = 300.0) -> float:
    """Demand (in chunks) the horizon cannot deliver: solve the phase-1 LP --
    same rows, final cumulative reads free in [0, u], maximise their sum --
    and return sum(u) minus its optimum (0 up to solver accuracy iff the
    reference's LP at this horizon is feasible). A phase-1 solve that does not
    converge raises SolverBackendError, like the reference's timed-out
    horizon probe (solver.py:160-161); its iterate is never a verdict."""
    from dataclasses import replace
    from .errors import SolverBackendError
    from .solver import OPTIMAL, SolverOptions, solve
    p1 = replace(plan, phase1=True, _desc=None)
    lp = build_from_plan(p1, device)
    try:
        sol = solve(lp, SolverOptions(eps_rel=eps_rel, max_iters=max_iters, time_limit=time_limit,
                                      device=device))
    finally:
        lp.close()
    if sol.status != OPTIMAL:
        raise SolverBackendError(f"phase-1 probe did not converge at K={plan.K} ({sol.status})")
    return float(plan.pair_units.sum() - sol.objective)


def horizon_feasible(plan: LpPlan, device: int = 0, max_iters: int = 2_000_000,
                     time_limit: float = 300.0) -> bool:
    """Phase-1 feasibility verdict: unmet demand above max(1e-3 chunk, 1e-6
    of the total) means infeasible. (solve() itself certifies infeasibility;
    this is the independent cross-check the tests use.)"""
    gap = feasibility_gap(plan, device, max_iters=max_iters, time_limit=time_limit)
    return gap <= max(1e-3, 1e-6 * float(plan.pair_units.sum()))
