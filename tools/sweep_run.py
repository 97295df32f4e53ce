"""configs[3]: epoch-duration x chunk-size sweep, 64 independent LPs, one
process per GPU. Launch with torchrun (--nproc-per-node N) or plain python.
Prints one JSON line (rank 0): LPs solved, max-over-ranks time, LPs/s."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2305_13479_b200.sweep import default_sweep, run_sweep, solve_instance  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
insts = default_sweep()
solve_instance(insts[0], device=local)  # warm-up: context, module load
if world > 1:
    dist.barrier()
t0 = time.perf_counter()
streams = int(os.environ.get("STREAMS", "8"))
recs = run_sweep(insts, rank, world, device=local, streams=streams)
el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
if world > 1:
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
if rank == 0:
    ok = sum(r["status"] == "optimal" for r in recs)
    print(json.dumps({"workload": "configs[3] sweep: 64 single-chassis NDv2 LPs (4 chunk sizes x 4 EM x 2 "
                      "collectives x 2 chunk counts)", "n_gpus": world, "streams_per_gpu": streams, "lps": len(recs), "optimal": ok,
                      "seconds_max_over_ranks": float(el), "lps_per_s": len(recs) / float(el),
                      "iters_total": sum(r["iters"] for r in recs)}), flush=True)
if world > 1:
    dist.destroy_process_group()
