"""NDv2 AllGather (1 chunk), slowest-link epochs, horizon 2 % above K*:
iterations and device time to 1e-4 (all three criteria) on one GPU for
growing chassis counts -- the trend the 32-chassis LP (configs[4]) follows."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, epoch_duration, generate_demand,  # noqa: E402
                                   make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

for ch in [int(v) for v in (sys.argv[1:] or ["4", "8", "16"])]:
    t = ndv2(ch)
    d = generate_demand("allgather", t, 1, 25000)
    tau = epoch_duration(t, 25000, "slowest", 1)
    K = int(round((64 * (ch - 1) + 3) * 1.02))
    lp = build_from_plan(make_plan(t, d, EpochConfig(tau, K, "slowest", 1, 25000)))
    for eps_res in (0.0, 1e-6):
        sol = solve(lp, SolverOptions(eps_rel=1e-4, eps_res=eps_res, time_limit=1800, max_iters=2_000_000))
        print(json.dumps({"chassis": ch, "K": K, "cols": lp.num_vars, "rows": lp.num_rows, "eps_res": eps_res,
                          "status": sol.status, "iters": sol.meta["iters"], "device_s": sol.meta["device_seconds"],
                          "ms_per_iter": 1e3 * sol.meta["device_seconds"] / max(1, sol.meta["iters"]),
                          "objective": sol.objective, "rel_gap": sol.meta["rel_gap"],
                          "rel_primal_res": sol.meta["rel_primal_res"]}), flush=True)
    lp.close()
