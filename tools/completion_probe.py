import sys, json, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2305_13479_b200 import *
from paper_2305_13479_b200.lp import build_from_plan
from paper_2305_13479_b200.topology import ndv2
for ch, K in ((1, 270), (2, 530)):
    t = ndv2(2); d = generate_demand("allgather", t, ch, 25000)
    tau = epoch_duration(t, 25000, "fastest", 1)
    plan = make_plan(t, d, EpochConfig(tau, K, "fastest", 1, 25000))
    lp = build_from_plan(plan)
    for eps in (1e-6, 1e-8, 1e-9):
        sol = solve(lp, SolverOptions(eps_rel=eps, max_iters=400000))
        rc = plan.rc_matrix(sol.x)
        short = plan.pair_units[:, None] - rc
        worst_pair_at = {k: float(short[:, k].max()) for k in (K-7, K-6, K-5, K-4, K-3, K-2)}
        rep = check_lp_schedule(plan, sol.x, tol=1e-5)
        print(ch, K, eps, sol.status, sol.meta["iters"], round(sol.meta["device_seconds"], 3), sol.objective,
              "comp", [lp_completion_epoch(sol, tol=tl) for tl in (1e-6, 1e-5, 1e-4)], "short", worst_pair_at,
              "check", rep.ok, rep.max_buffer_deficit, rep.max_capacity_excess, flush=True)
