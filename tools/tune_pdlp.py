"""Sweep PDLP restart / primal-weight / reflection parameters over a few
TE-CCL LPs; prints iterations and device seconds per (params, instance)."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, epoch_duration, generate_demand,  # noqa
                                   make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa
from paper_2305_13479_b200.topology import dgx2, ndv2  # noqa


def inst(kind, ch, K, topo):
    t = topo
    d = generate_demand(kind, t, ch, 25000)
    tau = epoch_duration(t, d.chunk_size, "fastest", 1)
    return build_from_plan(make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size)))


insts = {"ag2_K530": inst("allgather", 2, 530, ndv2(2)), "ag2_K520": inst("allgather", 2, 520, ndv2(2)),
         "ag2_K544": inst("allgather", 2, 544, ndv2(2)), "ag1_K270": inst("allgather", 1, 270, ndv2(2)),
         "ag1x4_K800": inst("allgather", 1, 800, ndv2(4)), "dgx2_a2a_K40": inst("alltoall", 1, 40, dgx2(1))}
grid = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
for params in grid:
    row = {"params": params}
    for name, lp in insts.items():
        sol = solve(lp, SolverOptions(eps_rel=1e-4, max_iters=200000, time_limit=30, pdlp=params))
        row[name] = (sol.meta["iters"], round(sol.meta["device_seconds"], 3), sol.status[:3])
    row["sum_s"] = round(sum(v[1] for k, v in row.items() if k not in ("params",)), 3)
    print(json.dumps(row), flush=True)
