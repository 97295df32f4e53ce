import sys, os
sys.path.insert(0, os.getcwd())
from paper_2305_13479_b200 import EpochConfig, SolverOptions, epoch_duration, generate_demand, make_plan, solve
from paper_2305_13479_b200.lp import build_from_plan
from paper_2305_13479_b200.topology import ndv2
t = ndv2(4); d = generate_demand("allgather", t, 1, 25000)
lp = build_from_plan(make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), 800, "fastest", 1, 25000)))
r = solve(lp, SolverOptions(eps_rel=1e-12, max_iters=1280))
print("OBJ", repr(r.objective), r.meta["iters"])
