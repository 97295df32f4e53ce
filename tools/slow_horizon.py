"""Smallest feasible horizon K* of NDv2 AllGather (1 chunk) with slowest-link
epochs for 2/4/8 chassis (device infeasibility certificates drive the
search): the chassis uplink / downlink carry 64 (chassis - 1) units at one
chunk per epoch, so K* = 64 (chassis - 1) + c; prints c per size."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, build_lp_model, epoch_duration,  # noqa: E402
                                   generate_demand, lp_completion_epoch, min_feasible_horizon)
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

for ch in [int(v) for v in (sys.argv[1:] or ["2", "4", "8"])]:
    t = ndv2(ch)
    d = generate_demand("allgather", t, 1, 25000)
    tau = epoch_duration(t, 25000, "slowest", 1)
    base = 64 * (ch - 1)
    t0 = time.perf_counter()
    k, sol = min_feasible_horizon(lambda K: build_lp_model(t, d, EpochConfig(tau, K, "slowest", 1, 25000)),
                                  base, base + 32, SolverOptions(eps_rel=1e-4, time_limit=900, max_iters=20_000_000))
    print(json.dumps({"chassis": ch, "K_star": k, "c": k - base, "search_s": time.perf_counter() - t0,
                      "objective": sol.objective, "iters": sol.meta["iters"],
                      "completion_epoch": lp_completion_epoch(sol, tol=1e-5)}), flush=True)
