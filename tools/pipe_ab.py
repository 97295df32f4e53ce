"""A/B of the pipelined half-step kernels on configs[1] (solve time, step bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
for cp in (0, 1):
    opts = SolverOptions(eps_rel=1e-4, pdlp={"col_pipeline": cp})
    for _ in range(2):
        s = solve(lp, opts)
    s8 = solve(lp, SolverOptions(eps_rel=1e-8, pdlp={"col_pipeline": cp}))
    print(cp, s.meta["iters"], round(s.meta["device_seconds"], 4),
          round(1e6 * s.meta["device_seconds"] / s.meta["iters"], 2), "us/it", s.objective,
          "| 1e-8:", s8.status, s8.meta["iters"], round(s8.meta["device_seconds"], 3), flush=True)
