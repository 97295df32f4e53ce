"""Row-partitioned single-LP solve across GPUs (north_star multi-GPU row).
torchrun --nproc-per-node N tools/dist_run.py [chassis] [chunks] [K] [eps] [compare]
Rank 0 prints one JSON line; with compare=1 it also solves the same LP on
one GPU and checks objective / finish time / integer replay of the gathered
partitioned solution."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2305_13479_b200 import (EpochConfig, SolverOptions, check_lp_schedule,  # noqa: E402
                                   epoch_duration, generate_demand, lp_completion_epoch,
                                   make_plan, solve)
from paper_2305_13479_b200.dist import solve_partitioned  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

chassis = int(sys.argv[1]) if len(sys.argv) > 1 else 2
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 2
K = int(sys.argv[3]) if len(sys.argv) > 3 else 530
eps = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-4
compare = int(sys.argv[5]) if len(sys.argv) > 5 else 1
max_iters = int(sys.argv[6]) if len(sys.argv) > 6 else 5_000_000
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, world = dist.get_rank(), dist.get_world_size()
assert torch.cuda.device_count() >= world, "one GPU per rank"
t = ndv2(chassis)
d = generate_demand("allgather", t, chunks, 25000)
cfg = EpochConfig(epoch_duration(t, d.chunk_size, "fastest", 1), K, "fastest", 1, d.chunk_size)
t0 = time.perf_counter()
pdlp = json.loads(os.environ.get("PDLP_OPTS", "{}"))  # e.g. '{"fused_halo": 0}'
out = solve_partitioned(t, d, cfg, eps_rel=eps, device=local, gather=bool(compare),
                        max_iters=max_iters, pdlp=pdlp)
wall = time.perf_counter() - t0
secs = torch.tensor([out["device_seconds"]], dtype=torch.float64, device=f"cuda:{local}")
dist.all_reduce(secs, op=dist.ReduceOp.MAX)
line = {"workload": f"ALLGATHER {chassis}-chassis NDv2, {chunks} chunk(s), K={K}, row-partitioned",
        "n_gpus": world, "eps_rel": eps, "status": out["status"], "iters": out["iters"],
        "objective": out["objective"], "device_seconds_max": float(secs), "wall_s": wall,
        "per_rank_epochs": [out["info"]["k0"], out["info"]["k1"]], "cols": out["info"]["total_cols"],
        "rows": out["info"]["total_rows"], "kernel_launches": out["kernel_launches"],
        "pdlp": pdlp}
if compare and rank == 0:
    plan = out["plan"]
    x = out["x"]
    class _S:  # solution-shaped record for lp_completion_epoch
        pass
    s = _S()
    s.x = x
    s.model = type("M", (), {"plan": plan})()
    line["completion_epoch"] = lp_completion_epoch(s, tol=1e-4)
    rep = check_lp_schedule(plan, x, tol=max(1e-5, 10 * eps), device=local)
    line["checker_ok"] = rep.ok
    single = solve(build_from_plan(plan, device=local), SolverOptions(eps_rel=eps, device=local))
    line["single_gpu"] = {"objective": single.objective, "iters": single.meta["iters"],
                          "device_seconds": single.meta["device_seconds"]}
    line["objective_rel_diff"] = abs(single.objective - out["objective"]) / abs(single.objective)
if rank == 0:
    print(json.dumps(line), flush=True)
dist.destroy_process_group()
