"""DGX-2 AllToAll family (configs[2]): smallest feasible horizon of the
2-chassis LP (device infeasibility certificates drive the search), and the
4-chassis LP one epoch below / at its K*, with timings."""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2305_13479_b200 import (EpochConfig, SolverOptions, build_lp_model, epoch_duration,  # noqa: E402
                                   generate_demand, lp_completion_epoch, min_feasible_horizon, solve)
from paper_2305_13479_b200.topology import dgx2  # noqa: E402


def fam(ch):
    t = dgx2(ch)
    d = generate_demand("alltoall", t, 1, 25000)
    return t, d, epoch_duration(t, 25000, "fastest", 1)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "2"
    if what == "2":
        t, d, tau = fam(2)
        t0 = time.perf_counter()
        k, sol = min_feasible_horizon(lambda K: build_lp_model(t, d, EpochConfig(tau, K, "fastest", 1, 25000)),
                                      200, 600, SolverOptions(time_limit=600, max_iters=10_000_000))
        print(json.dumps({"chassis": 2, "K_star": k, "search_s": time.perf_counter() - t0,
                          "objective": sol.objective, "iters": sol.meta["iters"],
                          "completion_epoch": lp_completion_epoch(sol, tol=1e-5)}), flush=True)
    else:
        t, d, tau = fam(4)
        for K, eps in ((1932, 1e-4), (1933, 1e-8)):
            lp = build_lp_model(t, d, EpochConfig(tau, K, "fastest", 1, 25000))
            sol = solve(lp, SolverOptions(eps_rel=eps, time_limit=900, max_iters=20_000_000))
            rec = {"chassis": 4, "K": K, "status": sol.status, "iters": sol.meta["iters"],
                   "device_s": sol.meta["device_seconds"], "cert": sol.meta["infeas_cert"],
                   "objective": sol.objective}
            if sol.feasible:
                rec["completion_epoch"] = lp_completion_epoch(sol, tol=1e-5)
                rec.update({k: sol.meta[k] for k in ("rel_gap", "rel_primal_res", "rel_dual_res",
                                                     "dual_objective")})
            print(json.dumps(rec), flush=True)
            lp.close()
