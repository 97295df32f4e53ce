"""Sweep PDLP parameters for time to the parity bar (gap 1e-4, residuals
1e-6) over several TE-CCL LPs; one JSON line per parameter set with the
iterations / device seconds per LP, their sum and the geometric mean of the
iteration ratios to the first set (usage: tune_parity.py '<json list>')."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, epoch_duration, generate_demand,  # noqa
                                   make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa
from paper_2305_13479_b200.topology import dgx2, ndv2  # noqa


def inst(kind, ch, K, t):
    d = generate_demand(kind, t, ch, 25000)
    tau = epoch_duration(t, d.chunk_size, "fastest", 1)
    return build_from_plan(make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size)))


insts = {"ag2_K530": inst("allgather", 2, 530, ndv2(2)), "ag2_K520": inst("allgather", 2, 520, ndv2(2)),
         "ag2_K544": inst("allgather", 2, 544, ndv2(2)), "ag1_K270": inst("allgather", 1, 270, ndv2(2)),
         "dgx2x2_K333": inst("alltoall", 1, 333, dgx2(2)), "dgx2_K40": inst("alltoall", 1, 40, dgx2(1)),
         "ag1x4_K800": inst("allgather", 1, 800, ndv2(4))}
grid = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
base = None
for params in grid:
    row = {"params": params}
    for name, lp in insts.items():
        sol = solve(lp, SolverOptions(max_iters=400000, time_limit=60, pdlp=params))
        row[name] = (sol.meta["iters"], round(sol.meta["device_seconds"], 3), sol.status[:3])
    its = {k: v[0] for k, v in row.items() if k != "params"}
    if base is None:
        base = its
    row["sum_s"] = round(sum(v[1] for k, v in row.items() if k != "params"), 3)
    row["geo"] = round(math.exp(sum(math.log(its[k] / base[k]) for k in its) / len(its)), 3)
    print(json.dumps(row), flush=True)
