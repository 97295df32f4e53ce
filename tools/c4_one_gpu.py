"""configs[4] (32-chassis NDv2 AllGather, slowest-link epochs, K=2024:
0.96e9 columns) solved on ONE B200 to the parity bar, with the integer-replay
certificate of the repaired flows. usage: python tools/c4_one_gpu.py [max_iters]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2305_13479_b200 import (EpochConfig, SolverOptions, check_lp_schedule, epoch_duration,  # noqa: E402
                                   generate_demand, make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan, completion_of  # noqa: E402
from paper_2305_13479_b200.schedule import max_deficit, repair_flows  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

max_iters = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
t = ndv2(32)
d = generate_demand("allgather", t, 1, 25000)
plan = make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "slowest", 1), 2024, "slowest", 1, 25000))
t0 = time.perf_counter()
lp = build_from_plan(plan)
build_s = time.perf_counter() - t0
pdlp = json.loads(os.environ.get("PDLP_OPTS", '{"step_safety": 0.9, "eps_infeas": 0.0, "verbose": 200}'))
sol = solve(lp, SolverOptions(max_iters=max_iters, time_limit=3300, pdlp=pdlp))
line = {"workload": "ALLGATHER 32-chassis NDv2, 1 chunk, slowest-link epochs, K=2024, one GPU",
        "cols": lp.num_vars, "rows": lp.num_rows, "status": sol.status, "build_s": build_s,
        "iters": sol.meta["iters"], "device_seconds": sol.meta["device_seconds"],
        "ms_per_iteration": 1e3 * sol.meta["device_seconds"] / max(1, sol.meta["iters"]),
        "objective": sol.objective, "rel_gap": sol.meta["rel_gap"],
        "rel_primal_res": sol.meta["rel_primal_res"], "rel_dual_res": sol.meta["rel_dual_res"], "pdlp": pdlp}
print(json.dumps(line), flush=True)
if sol.x is not None:
    lp.close()
    x = sol.x
    line = {"raw_max_pool_deficit": max_deficit(plan, x)}
    xr = repair_flows(plan, x)
    line["repaired_read_shortfall"] = float((plan.pair_units - plan.rd_matrix(xr).sum(axis=1)).max())
    rep = check_lp_schedule(plan, xr, tol=1e-3)
    line["checker_tol0.001"] = {"ok": rep.ok, "capacity_violations": rep.capacity_violations,
                                "causality_violations": rep.causality_violations,
                                "switch_violations": rep.switch_violations, "unmet_pairs": rep.unmet_pairs,
                                "completion_epoch": rep.completion_epoch}
    line["completion_epoch_tol0.001"] = completion_of(plan, xr, tol=1e-3)
    print(json.dumps(line), flush=True)
