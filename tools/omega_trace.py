"""Primal-weight trajectory of one solve (verbose PDLP log)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

cp, eps = int(sys.argv[1]), float(sys.argv[3])
extra = eval(sys.argv[4]) if len(sys.argv) > 4 else {}
t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
s = solve(lp, SolverOptions(eps_rel=eps, max_iters=400000, pdlp={"col_pipeline": cp, **extra}),
          verbose=int(sys.argv[5]) if len(sys.argv) > 5 else 50)
print(s.status, s.meta["iters"], s.meta["device_seconds"])
