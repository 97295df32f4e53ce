"""Short config-1 solve for ncu captures: builds the bench LP and runs a
bounded number of PDLP iterations (default 1280)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1280
t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
pdlp = json.loads(os.environ.get("PDLP_OPTS", "{}"))  # e.g. '{"matrix_free": 3}'
sol = solve(lp, SolverOptions(eps_rel=1e-12, max_iters=iters, time_limit=60, pdlp=pdlp))
print("iters", sol.meta["iters"], "status", sol.status, "device_s", sol.meta["device_seconds"])
