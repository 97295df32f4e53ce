"""A/B: the persistent chunk kernel vs the two-kernel iteration on configs[1]
(and a DGX-2 golden): iterations, device seconds, bit-identical iterates."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, epoch_duration, generate_demand,  # noqa: E402
                                   make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import dgx2, ndv2  # noqa: E402


def lp_of(t, kind, ch, K):
    d = generate_demand(kind, t, ch, 25000)
    tau = epoch_duration(t, 25000, "fastest", 1)
    return build_from_plan(make_plan(t, d, EpochConfig(tau, K, "fastest", 1, 25000)))


for name, lp in (("configs1", lp_of(ndv2(2), "allgather", 2, 530)), ("dgx2x1_K20", lp_of(dgx2(1), "alltoall", 1, 20))):
    res = {}
    for p in (0, 1, 0, 1):
        sol = solve(lp, SolverOptions(pdlp={"persist": p}))
        res.setdefault(p, []).append(sol)
        print(json.dumps({"lp": name, "persist": p, "iters": sol.meta["iters"], "s": sol.meta["device_seconds"],
                          "obj": sol.objective, "launches": sol.meta["kernel_launches"]}), flush=True)
    a, b = res[0][-1], res[1][-1]
    print(json.dumps({"lp": name, "identical_x": bool(np.array_equal(a.x, b.x)),
                      "identical_y": bool(np.array_equal(a.y, b.y)), "max_dx": float(np.abs(a.x - b.x).max())}),
          flush=True)
