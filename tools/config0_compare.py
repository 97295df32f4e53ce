"""configs[0]: ALLGATHER on single-chassis NDv2 (8 GPUs, 1 chunk/GPU), the
reference's CPU-runnable case. The reference's own LP path (its model
restated loop for loop by the oracle + the same scipy milp/HiGHS call) vs
this engine, on the same LP, at the smallest feasible horizon K* and at 2K*
and 4K* (or the horizons in argv[2], comma-separated). Prints one JSON line
per horizon.  usage: config0_compare.py [REF_TIME_LIMIT_S] [K,K,...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lp_oracle  # noqa: E402  (checker / reference arm only)
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, build_lp_model, epoch_duration,  # noqa: E402
                                   generate_demand, lp_completion_epoch, make_plan, min_feasible_horizon,
                                   solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

t = ndv2(1)
d = generate_demand("allgather", t, 1, 25000)
tau = epoch_duration(t, 25000, "fastest", 1)
cfg = EpochConfig(tau, 1, "fastest", 1, 25000)
kstar, _ = min_feasible_horizon(lambda K: build_lp_model(t, d, cfg.with_horizon(K)), 1, 256,
                                SolverOptions(eps_rel=1e-8))
tl = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
Ks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [kstar, 2 * kstar, 4 * kstar]
for K in Ks:
    out = {"workload": f"configs[0] ALLGATHER 1-chassis NDv2, 1 chunk, K={K}", "K_star": kstar}
    t0 = time.perf_counter()
    a = lp_oracle.build_lp_arrays(t, d, tau, K, 25000)
    out["ref_build_s"] = time.perf_counter() - t0
    r = lp_oracle.solve_highs(a, time_limit=tl)
    out.update({"ref_status": r["status"], "ref_solve_s": r["seconds"], "ref_objective": r.get("objective"),
                "rows": len(a["row_lo"]), "cols": len(a["var_lb"])})
    if r["status"] == "optimal":
        out["ref_completion_epoch"] = lp_oracle.completion_epoch(a, r["x"])
    for eps in (1e-4, 1e-8):
        plan = make_plan(t, d, cfg.with_horizon(K))
        build_from_plan(plan).close()  # warm-up
        t0 = time.perf_counter()
        lp = build_from_plan(make_plan(t, d, cfg.with_horizon(K)))
        sol = solve(lp, SolverOptions(eps_rel=eps))
        wall = time.perf_counter() - t0
        o = {"status": sol.status, "device_s": sol.meta["device_seconds"], "e2e_s": wall,
             "iters": sol.meta["iters"], "objective": sol.objective,
             "completion_epoch": lp_completion_epoch(sol, tol=1e-5)}
        if r["status"] == "optimal":
            o["objective_rel_err"] = abs(sol.objective - r["objective"]) / abs(r["objective"])
            o["speedup_e2e_vs_ref"] = (out["ref_build_s"] + r["seconds"]) / wall
        out[f"b200_eps_{eps:g}"] = o
        lp.close()
    print(json.dumps(out), flush=True)
