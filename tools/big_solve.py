"""Solve one large NDv2 AllGather LP on one GPU to eps and check it:
iterations, device seconds, objective, finish epoch, integer replay.
usage: python tools/big_solve.py CHASSIS K [EPS] [TIME_LIMIT_S]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, check_lp_schedule, epoch_duration,  # noqa: E402
                                   generate_demand, lp_completion_epoch, make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

ch, K = int(sys.argv[1]), int(sys.argv[2])
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
tl = float(sys.argv[4]) if len(sys.argv) > 4 else 3600.0
t = ndv2(ch)
d = generate_demand("allgather", t, 1, 25000)
plan = make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), K, "fastest", 1, 25000))
t0 = time.perf_counter()
lp = build_from_plan(plan)
build_s = time.perf_counter() - t0
sol = solve(lp, SolverOptions(eps_rel=eps, time_limit=tl, max_iters=50_000_000))
out = {"workload": f"ALLGATHER {ch}-chassis NDv2, 1 chunk, K={K}", "cols": lp.num_vars, "rows": lp.num_rows,
       "nnz": lp.nnz, "build_s": build_s, "eps_rel": eps, "status": sol.status, "iters": sol.meta["iters"],
       "restarts": sol.meta["restarts"], "device_seconds": sol.meta["device_seconds"],
       "ms_per_iter": 1e3 * sol.meta["device_seconds"] / max(1, sol.meta["iters"]),
       "objective": sol.objective, "rel_gap": sol.meta["rel_gap"],
       "rel_primal_res": sol.meta["rel_primal_res"], "rel_dual_res": sol.meta["rel_dual_res"]}
if sol.status == "optimal":
    out["completion_epoch"] = lp_completion_epoch(sol, tol=1e-3)
    rep = check_lp_schedule(plan, sol.x, tol=max(1e-4, 10 * eps))
    out["checker_ok"] = rep.ok
print(json.dumps(out), flush=True)
