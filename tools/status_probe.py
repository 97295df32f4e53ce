"""Probe: solve statuses / iterations of the infeasible goldens, a near-K*
infeasible horizon, and configs[1] at the parity bar vs the 1e-4 KKT point."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2305_13479_b200 import (EpochConfig, SolverOptions, epoch_duration, generate_demand,  # noqa: E402
                                   make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import dgx1, ndv2  # noqa: E402

KEYS = ("iters", "device_seconds", "rel_gap", "rel_primal_res", "rel_dual_res", "infeas_cert", "restarts")


def run(tag, t, d, K, **kw):
    tau = epoch_duration(t, d.chunk_size, "fastest", 1)
    lp = build_from_plan(make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size)))
    sol = solve(lp, SolverOptions(time_limit=120, max_iters=kw.pop("max_iters", 400_000), **kw))
    rec = {"tag": tag, "K": K, "status": sol.status, "objective": sol.objective}
    rec.update({k: sol.meta[k] for k in KEYS})
    print(json.dumps(rec), flush=True)
    lp.close()


if __name__ == "__main__":
    t1 = dgx1()
    ag1 = generate_demand("allgather", t1, 1, 25000)
    for K in (4, 6, 7, 8):
        run("dgx1_ag1", t1, ag1, K)
    t2 = ndv2(2)
    ag = generate_demand("allgather", t2, 1, 25000)
    for K in (24, 200):
        run("ndv2x2_ag1", t2, ag, K)
    ag2 = generate_demand("allgather", t2, 2, 25000)
    run("configs1_parity", t2, ag2, 530)
    run("configs1_kkt1e-4", t2, ag2, 530, eps_res=0.0)
    run("configs1_1e-8", t2, ag2, 530, eps_rel=1e-8)
    for K in (260, 500, 518):
        run("configs1_infeasible_probe", t2, ag2, K)
