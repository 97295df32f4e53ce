"""A/B of the stored-operator column kernels on configs[1]: col_pipe
(col_pipeline = 1) vs the two-columns-per-thread col_pipe2 (2): step-bench
time per launch and a full solve to the parity bar."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import (EpochConfig, SolverOptions, epoch_duration, generate_demand,  # noqa: E402
                                   make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

t = ndv2(2)
d = generate_demand("allgather", t, 2, 25000)
lp = build_from_plan(make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), 530, "fastest", 1, 25000)))
for cp in (1, 2, 1, 2):
    sb = min((lp.step_bench(400, {"col_pipeline": cp}) for _ in range(3)), key=lambda r: r["ms_col"])
    sol = solve(lp, SolverOptions(pdlp={"col_pipeline": cp}))
    print(json.dumps({"col_pipeline": cp, "us_col": 1e3 * sb["ms_col"], "us_row": 1e3 * sb["ms_row"],
                      "iters": sol.meta["iters"], "s": sol.meta["device_seconds"],
                      "us_per_iter": 1e6 * sol.meta["device_seconds"] / sol.meta["iters"],
                      "objective": sol.objective}), flush=True)
