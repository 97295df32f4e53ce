"""configs[2]: AllToAll on 4-chassis DGX-2 (64 GPUs + 4 switches; 125 GB/s
switch links alpha 0.35 us, 12.5 GB/s cross links alpha 2.6 us), fastest-link
epochs. Finds the smallest feasible horizon by phase-1 solves, then solves the
LP there to 1e-4 and 1e-8 and checks the schedule."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, check_lp_schedule, epoch_duration,  # noqa: E402
                                   generate_demand, lp_completion_epoch, make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan, feasibility_gap  # noqa: E402
from paper_2305_13479_b200.topology import dgx2  # noqa: E402

t = dgx2(4)
d = generate_demand("alltoall", t, 1, 25000)
tau = epoch_duration(t, d.chunk_size, "fastest", 1)
cfg0 = EpochConfig(tau, 8, "fastest", 1, d.chunk_size)
lo, hi = int(sys.argv[1]), int(sys.argv[2])
probes = {}
while lo < hi:  # smallest K with zero unmet demand
    mid = (lo + hi) // 2
    t0 = time.perf_counter()
    gap = feasibility_gap(make_plan(t, d, cfg0.with_horizon(mid)), eps_rel=1e-6)
    probes[mid] = (gap, time.perf_counter() - t0)
    print("probe", mid, probes[mid], flush=True)
    if gap <= 1e-3:
        hi = mid
    else:
        lo = mid + 1
K = lo
plan = make_plan(t, d, cfg0.with_horizon(K))
lp = build_from_plan(plan)
out = {"K_min": K, "tau_s": tau, "rows": lp.num_rows, "cols": lp.num_vars, "nnz": lp.nnz, "probes": probes}
for eps in (1e-4, 1e-8):
    sol = solve(lp, SolverOptions(eps_rel=eps, time_limit=1200, max_iters=5_000_000))
    out[f"eps_{eps:g}"] = {"status": sol.status, "iters": sol.meta["iters"],
                           "device_s": sol.meta["device_seconds"], "objective": sol.objective}
    if sol.status == "optimal":
        out[f"eps_{eps:g}"]["completion_epoch"] = lp_completion_epoch(sol, tol=1e-5)
out["checker_ok_1e-8"] = check_lp_schedule(plan, sol.x, tol=1e-5).ok
print(json.dumps(out), flush=True)
