"""One LP across GPUs partitioned by source (commodity):
torchrun --nproc-per-node N tools/src_run.py [chassis] [chunks] [K] [eps] [compare] [max_iters]
Rank 0 prints one JSON line; compare=1 also solves the LP on one GPU and
checks objective / finish time / integer replay of the gathered solution."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2305_13479_b200 import (EpochConfig, SolverOptions, check_lp_schedule,  # noqa: E402
                                   epoch_duration, generate_demand, lp_completion_epoch, make_plan, solve)
from paper_2305_13479_b200.dist import solve_source_partitioned  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import dgx2, ndv2  # noqa: E402

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
# TOPO=dgx2 COLL=alltoall for configs[2]-style LPs (default NDv2 AllGather)
topo = os.environ.get("TOPO", "ndv2")
coll = os.environ.get("COLL", "allgather")
t = {"ndv2": ndv2, "dgx2": dgx2}[topo](chassis)
d = generate_demand(coll, t, chunks, 25000)
cfg = EpochConfig(epoch_duration(t, d.chunk_size, "fastest", 1), K, "fastest", 1, d.chunk_size)
t0 = time.perf_counter()
out = solve_source_partitioned(t, d, cfg, eps_rel=eps, device=local, gather=bool(compare), max_iters=max_iters)
wall = time.perf_counter() - t0
secs = torch.tensor([out["device_seconds"]], dtype=torch.float64, device=f"cuda:{local}")
dist.all_reduce(secs, op=dist.ReduceOp.MAX)
line = {"workload": f"{coll.upper()} {chassis}-chassis {topo}, {chunks} chunk(s), K={K}, source-partitioned",
        "n_gpus": world, "eps_rel": eps, "status": out["status"], "iters": out["iters"],
        "objective": out["objective"], "device_seconds_max": float(secs), "wall_s": wall,
        "rel_gap": out["rel_gap"], "info": out["info"]}
if compare and rank == 0:
    plan = out["plan"]

    class _S:
        pass
    s = _S()
    s.x = out["x"]
    s.model = type("M", (), {"plan": plan})()
    line["completion_epoch"] = lp_completion_epoch(s, tol=1e-4)
    single = solve(build_from_plan(plan, device=local), SolverOptions(eps_rel=eps, device=local,
                                                                      max_iters=max_iters))
    line["single_gpu"] = {"objective": single.objective, "iters": single.meta["iters"],
                          "device_seconds": single.meta["device_seconds"]}
    line["objective_rel_diff"] = abs(single.objective - out["objective"]) / abs(single.objective)
    if eps <= 1e-7:
        line["checker_ok"] = check_lp_schedule(plan, out["x"], tol=1e-5, device=local).ok
if rank == 0:
    print(json.dumps(line), flush=True)
dist.destroy_process_group()
