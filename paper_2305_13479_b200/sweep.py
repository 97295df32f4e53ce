"""Independent-instance sweeps, one process per GPU (configs[3]).

Epoch-duration x chunk-size sweeps and multi-demand batches are independent
LPs: each rank solves its own shard on its own GPU, with no data-path
collective; only the small per-instance result records are gathered at the
end (torch.distributed all_gather_object, NCCL or gloo). Mirrors how the
reference's workflow would be looped over parameters (workflow.py:39-113),
with the LP solve moved to the GPU.
"""

from __future__ import annotations

import itertools
import time
from dataclasses import asdict, dataclass

from .demand import generate_demand
from .epochs import EpochConfig, epoch_duration
from .topology import dgx1, dgx2, ndv2


@dataclass(frozen=True)
class Instance:
    topology: str          # "ndv2" | "dgx1" | "dgx2"
    chassis: int
    collective: str        # "allgather" | "alltoall"
    chunks: int
    chunk_size: int        # bytes
    em: int                # epoch multiplier
    K: int


def default_sweep() -> list[Instance]:
    """64 LPs: single-chassis NDv2, 4 chunk sizes x 4 epoch multipliers x
    2 collectives x 2 chunk counts, all at a horizon comfortably above the
    minimum feasible one."""
    out = []
    for size, em, coll, ch in itertools.product((25_000, 50_000, 100_000, 200_000), (1, 2, 3, 4),
                                                ("allgather", "alltoall"), (1, 2)):
        out.append(Instance("ndv2", 1, coll, ch, size, em, 24 * ch))
    return out


def shard(items: list, rank: int, world: int) -> list:
    """Round-robin shard: rank r takes items r, r+world, ... (deterministic)."""
    return items[rank::world]


def build_instance(inst: Instance):
    gen = {"ndv2": ndv2, "dgx1": lambda chassis=1: dgx1(), "dgx2": dgx2}[inst.topology]
    t = gen(chassis=inst.chassis)
    d = generate_demand(inst.collective, t, inst.chunks, inst.chunk_size)
    tau = epoch_duration(t, d.chunk_size, "fastest", inst.em)
    return t, d, EpochConfig(tau, inst.K, "fastest", inst.em, d.chunk_size)


def solve_instance(inst: Instance, device: int = 0, eps_rel: float = 1e-4, slot: int = 0) -> dict:
    from .lp import build_lp_model, lp_completion_epoch
    from .solver import SolverOptions, solve
    t, d, cfg = build_instance(inst)
    t0 = time.perf_counter()
    lp = build_lp_model(t, d, cfg, device=device, slot=slot)
    sol = solve(lp, SolverOptions(eps_rel=eps_rel, device=device))
    rec = {"instance": asdict(inst), "status": sol.status, "objective": sol.objective,
           "iters": sol.meta["iters"], "device_seconds": sol.meta["device_seconds"],
           "wall_seconds": time.perf_counter() - t0, "tau": cfg.tau}
    try:
        comp = lp_completion_epoch(sol, tol=1e-4)
        rec["completion_epoch"] = comp
        rec["finish_time_s"] = (comp + 1) * cfg.tau
    except Exception as exc:  # a horizon too short for the demand
        rec["completion_epoch"] = None
        rec["error"] = str(exc)
    lp.close()
    return rec


def solve_shard(items: list, device: int, solver, streams: int = 1) -> list:
    """Solve (index, instance) pairs on one GPU. streams > 1: that many host
    threads, each driving its own context (CUDA stream) on the device, take
    instances from a shared queue -- small LPs are launch/latency-bound, so
    concurrent solves fill the GPU that one solve leaves idle. Records come
    back in input order."""
    if streams <= 1 or len(items) <= 1:
        return [(i, solver(inst, device)) for i, inst in items]
    import queue
    import threading
    q = queue.Queue()
    for it in items:
        q.put(it)
    out, errs = {}, []

    def work(slot):
        while True:
            try:
                i, inst = q.get_nowait()
            except queue.Empty:
                return
            try:
                out[i] = solver(inst, device, slot=slot)
            except Exception as exc:  # surfaced after the join
                errs.append(exc)
                return

    threads = [threading.Thread(target=work, args=(k,)) for k in range(min(streams, len(items)))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return [(i, out[i]) for i, _ in items]


def run_sweep(instances: list[Instance], rank: int = 0, world: int = 1, device: int = 0,
              solver=solve_instance, group=None, streams: int = 1) -> list[dict]:
    """Solve this rank's shard (`streams` concurrent solves on the rank's
    GPU); with world > 1 gather every record on every rank (ordered like
    `instances`)."""
    mine = solve_shard(list(zip(range(rank, len(instances), world), shard(instances, rank, world))),
                       device, solver, streams)
    if world == 1:
        return [r for _, r in mine]
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    merged = sorted((pair for part in parts for pair in part), key=lambda p: p[0])
    return [r for _, r in merged]
