import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload
from paper_2305_13479_b200 import SolverOptions, make_plan, solve
from paper_2305_13479_b200.lp import build_from_plan
t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
for its in (64, 128):
    res = {}
    for cp in (0, 1):
        s = solve(lp, SolverOptions(eps_rel=1e-12, max_iters=its, pdlp={"col_pipeline": cp}))
        res[cp] = s
    print(its, "x diff", float(np.abs(res[0].x - res[1].x).max()), "y diff", float(np.abs(res[0].y - res[1].y).max()),
          "omega", res[0].meta["omega"], res[1].meta["omega"], "restarts", res[0].meta["restarts"], res[1].meta["restarts"], flush=True)
