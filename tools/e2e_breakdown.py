"""Where the e2e time goes: host plan, device build (+SELL), solve, D2H."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, check_lp_schedule, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

t, d, cfg = workload()
for rep in range(3):
    t0 = time.perf_counter()
    plan = make_plan(t, d, cfg)
    t1 = time.perf_counter()
    lp = build_from_plan(plan)
    t2 = time.perf_counter()
    sol = solve(lp, SolverOptions(eps_rel=1e-4))
    t3 = time.perf_counter()
    print(f"plan {t1-t0:.4f}s build {t2-t1:.4f}s solve_wall {t3-t2:.4f}s device {sol.meta['device_seconds']:.4f}s", flush=True)
    lp.close()
sol6 = solve(build_from_plan(plan), SolverOptions(eps_rel=1e-6))
for tol in (1e-6, 1e-5, 1e-4, 1e-3):
    print(tol, check_lp_schedule(plan, sol6.x, tol=tol))
