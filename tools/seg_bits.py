"""Fixed-iteration solve of the 4-chassis LP on the large-LP operator (mode 4:
col_te2 + row_seg): prints the objective and a hash of x, so two builds of the
row kernel can be compared bit for bit."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import EpochConfig, SolverOptions, epoch_duration, generate_demand, make_plan, solve  # noqa
from paper_2305_13479_b200.lp import build_from_plan  # noqa
from paper_2305_13479_b200.topology import ndv2  # noqa

t = ndv2(4)
d = generate_demand("allgather", t, 1, 25000)
lp = build_from_plan(make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), 800, "fastest", 1, 25000)))
sol = solve(lp, SolverOptions(eps_rel=1e-12, eps_res=0.0, max_iters=1280, pdlp={"matrix_free": 4}))
print(json.dumps({"lib": os.environ.get("TECCL_B200_LIB", "default"), "iters": sol.meta["iters"],
                  "objective": sol.objective, "x_sha": hashlib.sha1(sol.x.tobytes()).hexdigest()[:16],
                  "y_sha": hashlib.sha1(sol.y.tobytes()).hexdigest()[:16]}))
