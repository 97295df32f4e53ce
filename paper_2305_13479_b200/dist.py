"""One LP row-partitioned by epoch block across GPUs (one process per GPU).

North-star row (e): a single large multi-chassis LP is split into
contiguous epoch blocks; rank r builds only its block (csrc/te_build.cu,
epoch-major numbering), the ranks exchange CUDA IPC handles of their
exchange arenas once through torch.distributed (NCCL or gloo), and the PDLP
iteration then moves the primal/dual halo vectors and the KKT scalars
through peer memory over NVLink inside the solve -- no host round trips.
Every rank takes identical restart/termination decisions because the global
sums are formed in rank order on every rank.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .lp import LpPlan, apply_operator, make_plan, step_bench

INFO_KEYS = ("own_c0", "own_c1", "own_r0", "own_r1", "win_c0", "win_c1", "win_r0", "win_r1",
             "k0", "k1", "total_cols", "total_rows", "delta_max", "nnz_csr", "nnz_csc",
             "cols_per_epoch")


@dataclass
class PartLP:
    handle: object
    ctx: nat.Context
    plan: LpPlan
    world: int
    rank: int
    info: dict

    def apply(self, v: np.ndarray, transpose: bool = False, matrix_free: int = 1) -> dict:
        """This block's rows of A.v (v over the column window) or columns of
        A^T.v (v over the row window), stored (0) or matrix-free (1) operator."""
        i = self.info
        nin = (i["win_r1"] - i["win_r0"]) if transpose else (i["win_c1"] - i["win_c0"])
        nout = (i["own_c1"] - i["own_c0"]) if transpose else (i["own_r1"] - i["own_r0"])
        return apply_operator(self.ctx, self.handle, v, nin, nout, transpose, matrix_free)

    def step_bench(self, reps: int = 50, pdlp: dict | None = None) -> dict:
        """Half-step kernel timing on this block (world = 1 blocks only: the
        kernels of a connected block wait for their neighbours)."""
        return step_bench(self.ctx, self.handle, reps, pdlp)

    def close(self):
        if self.handle:
            self.ctx.lib.teccl_lp_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_partition(plan: LpPlan, world: int, rank: int, device: int = 0) -> PartLP:
    ctx = nat.Context.get(device)
    h = C.c_void_p()
    info = (C.c_int64 * 16)()
    nat.check(ctx.lib.teccl_lp_build_te_part(ctx.handle, C.byref(plan.desc()), int(world),
                                             int(rank), C.byref(h), info))
    return PartLP(h, ctx, plan, world, rank, dict(zip(INFO_KEYS, list(info))))


def export_blob(part: PartLP) -> bytes:
    buf = (C.c_uint8 * 512)()
    n = C.c_int64()
    nat.check(part.ctx.lib.teccl_dist_export(part.ctx.handle, part.handle, buf, C.byref(n)))
    return bytes(buf[:n.value])


def connect(part: PartLP, blobs: list[bytes]) -> None:
    if len(blobs) != part.world or len({len(b) for b in blobs}) != 1:
        raise ValueError("need one blob per rank, all the same length")
    joined = b"".join(blobs)
    arr = (C.c_uint8 * len(joined)).from_buffer_copy(joined)
    nat.check(part.ctx.lib.teccl_dist_connect(part.ctx.handle, part.handle, arr, len(blobs[0])))


def em_to_ref_cols(plan: LpPlan, c0: int, c1: int) -> np.ndarray:
    """Reference column index of epoch-major columns [c0, c1) (te_build.cu
    ref_col_of_em, vectorised)."""
    S, E, G, P, K = plan.S, plan.E, plan.G, plan.P, plan.K
    SB = plan.SB
    CW = S * E + S * G + 2 * P
    c = np.arange(c0, c1, dtype=np.int64)
    k = c // CW
    o = c - k * CW
    out = np.empty_like(c)
    tail = k >= K
    o2 = c[tail] - K * CW
    out[tail] = (o2 // G) * SB + E * K + (o2 % G) * (K + 1) + K
    body = ~tail
    kb, ob = k[body], o[body]
    res = np.empty_like(kb)
    f = ob < S * E
    res[f] = (ob[f] // E) * SB + (ob[f] % E) * K + kb[f]
    b = (~f) & (ob < S * E + S * G)
    ob2 = ob[b] - S * E
    res[b] = (ob2 // G) * SB + E * K + (ob2 % G) * (K + 1) + kb[b]
    r = (~f) & (~b)
    ob3 = ob[r] - S * E - S * G
    res[r] = S * SB + (ob3 // 2) * 2 * K + 2 * kb[r] + (ob3 % 2)
    out[body] = res
    return out


def partition_epochs(K: int, world: int) -> list[tuple[int, int]]:
    """Epoch block of every rank (same split as teccl_lp_build_te_part)."""
    return [(r * K // world, (r + 1) * K // world) for r in range(world)]


def solve_partitioned(t, d, cfg, opts=None, eps_rel: float = 1e-4, max_iters: int = 5_000_000,
                      eps_res: float = 1e-6,
                      device: int | None = None, group=None, gather: bool = False,
                      pdlp: dict | None = None) -> dict:
    """Collective call: every rank of the process group solves its epoch
    block; returns the (identical) global status/objective on every rank and,
    with gather=True, the full solution in reference column order on rank 0
    (gather="all": on every rank)."""
    import torch
    import torch.distributed as dist
    from .solver import SolverOptions, pdlp_options
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if device is None:
        device = torch.cuda.current_device()
    plan = make_plan(t, d, cfg, opts)
    if world == 1:  # nothing to partition: the single-device path
        from .lp import build_from_plan
        from .solver import solve
        lp = build_from_plan(plan, device)
        sol = solve(lp, SolverOptions(eps_rel=eps_rel, eps_res=eps_res, max_iters=max_iters, device=device,
                                      pdlp=pdlp or {}))
        out = {"status": sol.status, "objective": sol.objective, "iters": sol.meta["iters"],
               "restarts": sol.meta["restarts"], "rel_gap": sol.meta["rel_gap"],
               "rel_primal_res": sol.meta["rel_primal_res"],
               "rel_dual_res": sol.meta["rel_dual_res"],
               "device_seconds": sol.meta["device_seconds"],
               "kernel_launches": sol.meta["kernel_launches"], "world": 1, "rank": 0,
               "info": {"own_c0": 0, "own_c1": plan.num_vars, "k0": 0, "k1": plan.K,
                        "total_cols": plan.num_vars, "total_rows": plan.num_rows}}
        if gather:
            out["x"] = sol.x
            out["plan"] = plan
        lp.close()
        return out
    part = build_partition(plan, world, rank, device)
    blobs = [None] * world
    dist.all_gather_object(blobs, export_blob(part), group=group)
    connect(part, blobs)
    dist.barrier(group=group)
    n_own = part.info["own_c1"] - part.info["own_c0"]
    m_own = part.info["own_r1"] - part.info["own_r0"]
    x = np.empty(max(1, n_own))
    y = np.empty(max(1, m_own))
    res = nat.PdlpResult()
    o = pdlp_options(SolverOptions(eps_rel=eps_rel, eps_res=eps_res, max_iters=max_iters, device=device,
                                   pdlp=pdlp or {}))
    nat.check(part.ctx.lib.teccl_pdlp_solve(part.ctx.handle, part.handle, C.byref(o),
                                            nat.ptr(x, C.c_double), nat.ptr(y, C.c_double),
                                            C.byref(res)))
    out = {"status": nat.STATUS.get(res.status, "peer-timeout" if res.status == 5 else "?"),
           "objective": -res.primal_obj, "iters": int(res.iters), "restarts": int(res.restarts),
           "rel_gap": res.rel_gap, "rel_primal_res": res.rel_primal_res,
           "rel_dual_res": res.rel_dual_res, "device_seconds": res.solve_seconds,
           "kernel_launches": int(res.spmv_launches), "world": world, "rank": rank,
           "info": part.info}
    if gather:  # the full solution on rank 0 (gather="all": on every rank)
        piece = (part.info["own_c0"], part.info["own_c1"], x[:n_own])
        pieces = [None] * world
        if gather == "all":
            dist.all_gather_object(pieces, piece, group=group)
        else:
            dist.gather_object(piece, pieces if rank == 0 else None, dst=0, group=group)
        if gather == "all" or rank == 0:
            full = np.empty(plan.num_vars)
            for c0, c1, xs in pieces:
                full[em_to_ref_cols(plan, c0, c1)] = xs
            out["x"] = full
        out["plan"] = plan
    part.close()
    return out


SRC_INFO_KEYS = ("s0", "s1", "p0", "p1", "c0", "c1", "q0", "q1")


def solve_source_partitioned(t, d, cfg, opts=None, eps_rel: float = 1e-4, max_iters: int = 5_000_000,
                             eps_res: float = 1e-6,
                             device: int | None = None, group=None, gather: bool = False,
                             pdlp: dict | None = None) -> dict:
    """Collective call: ONE LP across the ranks of the group, partitioned by
    source (commodity). Every rank builds the whole LP on its GPU and runs the
    (identical) setup; in the iteration rank r updates the flows, buffers and
    reads of sources [s0, s1) and their rows, and the capacity rows -- the only
    rows shared by the commodities -- are summed across ranks every iteration
    through peer memory (csrc/pdlp.cu cap_part_kernel / cap_fin_kernel).
    Returns the (identical) status / objective on every rank and, with
    gather=True, the full solution in reference column order."""
    import torch
    import torch.distributed as dist
    from .lp import build_from_plan
    from .solver import SolverOptions, pdlp_options
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if device is None:
        device = torch.cuda.current_device()
    plan = make_plan(t, d, cfg, opts)
    lp = build_from_plan(plan, device)
    info = (C.c_int64 * 8)()
    nat.check(lp.ctx.lib.teccl_src_setup(lp.ctx.handle, lp.handle, int(world), int(rank), info))
    info = dict(zip(SRC_INFO_KEYS, list(info)))
    buf = (C.c_uint8 * 512)()
    blen = C.c_int64()
    nat.check(lp.ctx.lib.teccl_src_export(lp.ctx.handle, lp.handle, buf, C.byref(blen)))
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes(buf[:blen.value]), group=group)
    joined = b"".join(blobs)
    arr = (C.c_uint8 * len(joined)).from_buffer_copy(joined)
    nat.check(lp.ctx.lib.teccl_src_connect(lp.ctx.handle, lp.handle, arr, blen.value))
    dist.barrier(group=group)
    x = np.empty(plan.num_vars)
    y = np.empty(plan.num_rows)
    res = nat.PdlpResult()
    o = pdlp_options(SolverOptions(eps_rel=eps_rel, eps_res=eps_res, max_iters=max_iters, device=device,
                                   pdlp=pdlp or {}))
    nat.check(lp.ctx.lib.teccl_pdlp_solve(lp.ctx.handle, lp.handle, C.byref(o),
                                          nat.ptr(x, C.c_double), nat.ptr(y, C.c_double),
                                          C.byref(res)))
    out = {"status": nat.STATUS.get(res.status, "peer-timeout" if res.status == 5 else "?"),
           "objective": -res.primal_obj, "iters": int(res.iters), "restarts": int(res.restarts),
           "rel_gap": res.rel_gap, "rel_primal_res": res.rel_primal_res,
           "rel_dual_res": res.rel_dual_res, "device_seconds": res.solve_seconds,
           "kernel_launches": int(res.spmv_launches), "world": world, "rank": rank,
           "info": dict(info, total_cols=plan.num_vars, total_rows=plan.num_rows)}
    if gather:  # the full solution on rank 0 (gather="all": on every rank)
        own = (info["c0"], info["c1"], x[info["c0"]:info["c1"]].copy(),
               info["q0"], info["q1"], x[info["q0"]:info["q1"]].copy())
        pieces = [None] * world
        if gather == "all":
            dist.all_gather_object(pieces, own, group=group)
        else:
            dist.gather_object(own, pieces if rank == 0 else None, dst=0, group=group)
        if gather == "all" or rank == 0:
            full = np.empty(plan.num_vars)
            for c0, c1, xa, q0, q1, xb in pieces:
                full[c0:c1] = xa
                full[q0:q1] = xb
            out["x"] = full
        out["plan"] = plan
    lp.close()
    return out


def solve_distributed(t, d, cfg, opts=None, scheme: str = "auto", **kw) -> dict:
    """One LP across the ranks of the group. scheme "source": partition by
    commodity (whole LP per rank, fastest while the LP fits one GPU);
    "epoch": epoch-block row partition (memory-scalable); "auto": "source"
    when the LP's indices fit the single-device 31-bit limit, else "epoch"."""
    if scheme == "auto":
        plan = make_plan(t, d, cfg, opts)
        scheme = "source" if max(plan.num_vars, plan.num_rows) < (1 << 31) - 1 else "epoch"
    if scheme == "source":
        return solve_source_partitioned(t, d, cfg, opts, **kw)
    if scheme == "epoch":
        return solve_partitioned(t, d, cfg, opts, **kw)
    raise ValueError(f"unknown scheme {scheme!r} (auto, source, epoch)")
