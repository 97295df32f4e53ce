"""configs[4]: ALLGATHER on 32-chassis NDv2 (256 GPUs + switch), ONE LP
row-partitioned by epoch block over the torchrun ranks (dist.solve_partitioned:
halos and KKT scalars through CUDA-IPC peer memory over NVLink).

  torchrun --nproc-per-node N tools/c4_solve.py [chassis] [K] [mode] [eps] [max_iters] [gather] [eps_res]

Rank 0 prints one JSON line: status, iterations, device time (max over
ranks), the KKT certificate (relative gap, primal and dual residuals), and
with gather=1 the certificate of the schedule: the gathered solution's flows
repaired to conserve exactly (schedule.repair_flows) and replayed by the
exact-integer GPU checker, with the finish epoch. PDLP_OPTS (JSON) overrides
raw teccl_pdlp_opts fields (e.g. '{"verbose": 50}')."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2305_13479_b200 import (EpochConfig, check_lp_schedule, epoch_duration,  # noqa: E402
                                   generate_demand)
from paper_2305_13479_b200.dist import solve_partitioned, solve_source_partitioned  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

chassis = int(sys.argv[1]) if len(sys.argv) > 1 else 32
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2024
mode = sys.argv[3] if len(sys.argv) > 3 else "slowest"
eps = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-4
max_iters = int(sys.argv[5]) if len(sys.argv) > 5 else 600_000
gather = int(sys.argv[6]) if len(sys.argv) > 6 else 1
eps_res = float(sys.argv[7]) if len(sys.argv) > 7 else 0.0   # 1e-6: the parity bar
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, world = dist.get_rank(), dist.get_world_size()
t = ndv2(chassis)
d = generate_demand("allgather", t, 1, 25000)
cfg = EpochConfig(epoch_duration(t, 25000, mode, 1), K, mode, 1, 25000)
pdlp = json.loads(os.environ.get("PDLP_OPTS", "{}"))
t0 = time.perf_counter()
scheme = os.environ.get("SCHEME", "epoch")  # "source": whole LP per rank, partitioned by source
fn = solve_source_partitioned if scheme == "source" else solve_partitioned
out = fn(t, d, cfg, eps_rel=eps, eps_res=eps_res, max_iters=max_iters, device=local,
         gather=bool(gather), pdlp=pdlp)
wall = time.perf_counter() - t0
secs = torch.tensor([out["device_seconds"]], dtype=torch.float64, device=f"cuda:{local}")
dist.all_reduce(secs, op=dist.ReduceOp.MAX)
line = {"workload": f"ALLGATHER {chassis}-chassis NDv2, 1 chunk, {mode}-link epochs, K={K}, "
                    f"{'by source' if scheme == 'source' else 'epoch blocks'} over {world} GPUs",
        "n_gpus": world, "eps_rel": eps, "eps_res": eps_res,
        "criterion": "gap <= eps_rel, primal and dual residuals <= min(eps_rel, eps_res) (eps_res 0: eps_rel)",
        "status": out["status"], "iters": out["iters"], "restarts": out["restarts"],
        "objective": out["objective"], "rel_gap": out["rel_gap"],
        "rel_primal_res": out["rel_primal_res"], "rel_dual_res": out["rel_dual_res"],
        "device_seconds_max": float(secs), "ms_per_iteration": 1e3 * float(secs) / max(1, out["iters"]),
        "wall_s": wall, "cols": out["info"]["total_cols"], "rows": out["info"]["total_rows"],
        "partition": {k: out["info"].get(k) for k in ("k0", "k1", "s0", "s1")}, "pdlp": pdlp}
if rank == 0 and gather:  # the solve's line first: certification below can take minutes
    print(json.dumps(line), flush=True)
if gather and rank == 0:
    import numpy as np
    from paper_2305_13479_b200.lp import completion_of
    from paper_2305_13479_b200.schedule import max_deficit, repair_flows
    plan = out["plan"]
    x = out["x"]
    t1 = time.perf_counter()
    line["raw_max_pool_deficit"] = max_deficit(plan, x)
    xr = repair_flows(plan, x)
    line["repaired_read_shortfall"] = float((plan.pair_units - plan.rd_matrix(xr).sum(axis=1)).max())
    for tol in (1e-5, 1e-3):  # chunk fractions of slack in the integer replay
        try:
            line[f"completion_epoch_tol{tol:g}"] = completion_of(plan, xr, tol=tol)
        except Exception as exc:  # a pair short of its demand by more than tol
            line[f"completion_epoch_tol{tol:g}"] = str(exc)
        rep = check_lp_schedule(plan, xr, tol=tol, device=local)
        line[f"checker_tol{tol:g}"] = {"ok": rep.ok, "capacity_violations": rep.capacity_violations,
                                        "causality_violations": rep.causality_violations,
                                        "switch_violations": rep.switch_violations,
                                        "unmet_pairs": rep.unmet_pairs, "completion_epoch": rep.completion_epoch}
    line["certify_host_s"] = time.perf_counter() - t1
    line["objective_repaired"] = float(np.dot(plan.rc_matrix(xr).sum(axis=0), 1.0 / np.arange(1, plan.K + 1)))
if rank == 0:
    print(json.dumps(line), flush=True)
dist.destroy_process_group()
