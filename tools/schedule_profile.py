"""Phase timings of lp_rates_to_schedule on configs[1] (deficit check, flow
repair, native decomposition, event objects) at eps 1e-4 and 1e-8."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, make_plan, solve  # noqa: E402
from paper_2305_13479_b200 import schedule as S  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

t, d, cfg = workload()
plan = make_plan(t, d, cfg)
lp = build_from_plan(plan)
for eps in (1e-4, 1e-8):
    sol = solve(lp, SolverOptions(eps_rel=eps))
    x = np.asarray(sol.x, dtype=np.float64)
    out = {"eps": eps}
    t0 = time.perf_counter(); dfc = S.max_deficit(plan, x); out["max_deficit_s"] = time.perf_counter() - t0
    out["deficit"] = dfc
    tol = S.TOL
    if dfc > S.RAW_OK:
        t0 = time.perf_counter(); x = S.repair_flows(plan, x); out["repair_s"] = time.perf_counter() - t0
        tol = S.DUST
    try:
        t0 = time.perf_counter(); ev = S.decompose_native(plan, x, tol); out["decompose_native_s"] = time.perf_counter() - t0
        out["events"] = len(ev)
    except Exception as exc:
        out["decompose_native_error"] = str(exc)[:120]
    t0 = time.perf_counter(); s2 = S.lp_rates_to_schedule(sol); out["total_s"] = time.perf_counter() - t0
    out["schedule_meta"] = s2.meta
    print(json.dumps(out), flush=True)
