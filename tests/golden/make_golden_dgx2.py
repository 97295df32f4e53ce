"""Full-size golden for the DGX-2 AllToAll family (configs[2]), from the
REFERENCE package: the 2-chassis LP (collsched.topology.dgx2(2), AllToAll, 1
chunk, fastest-link epochs) at its smallest feasible horizon K* = 333 (found
on the GPU by min_feasible_horizon, profiles/r02_c_dgx2x2_horizon.log) built by
collsched.lp.build_lp_model and solved with HiGHS (interior point +
crossover, as make_golden_full.py), and K* - 1 = 332 whose status pins the
device's infeasibility certificate. Writes full_size_dgx2.json. Takes about
an hour on an 8-core host:
    python tests/golden/make_golden_dgx2.py
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from collsched import generate_demand  # noqa: E402
from collsched.epochs import EpochConfig, epoch_duration  # noqa: E402
from collsched.lp import build_lp_model, lp_completion_epoch  # noqa: E402
from collsched.milp import ModelOptions  # noqa: E402
from collsched.solver import OPTIMAL, Solution  # noqa: E402
from collsched.topology import dgx2  # noqa: E402

from make_golden_full import solve_ipm  # noqa: E402


def main():
    out = {}
    path = os.path.join(HERE, "full_size_dgx2.json")
    for K in (333, 332):
        t = dgx2(2)
        d = generate_demand("alltoall", t, 1, 25000)
        tau = epoch_duration(t, d.chunk_size, "fastest", 1)
        t0 = time.time()
        m = build_lp_model(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size), ModelOptions())
        build_s = time.time() - t0
        res, secs = solve_ipm(m)
        rec = {"chassis": 2, "kind": "alltoall", "chunks": 1, "K": K, "status": int(res.status),
               "message": str(res.message), "highs_ipm_seconds": secs, "reference_build_seconds": build_s,
               "num_vars": m.num_vars, "num_rows": len(m.rows)}
        if res.status == 0:
            sol = Solution(OPTIMAL, m, np.asarray(res.x), float(-res.fun))
            rec.update({"objective": float(-res.fun), "completion_epoch": lp_completion_epoch(sol)})
        out[f"dgx2x2_a2a1_K{K}"] = rec
        print(rec, flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main()
