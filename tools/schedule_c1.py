"""configs[1]: GPU solve to 1e-8, rate->schedule decomposition, replay with the
reference simulator restatement; prints timings and the verdict."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from oracle.simulator import simulate  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, lp_rates_to_schedule, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

t, d, cfg = workload()
plan = make_plan(t, d, cfg)
sol = solve(build_from_plan(plan), SolverOptions(eps_rel=1e-8))
t0 = time.perf_counter()
sched = lp_rates_to_schedule(sol)
t1 = time.perf_counter()
ev = [(e.source, e.chunk, e.src, e.dst, e.epoch, e.fraction) for e in sched.events]
rep = simulate(ev, cfg.tau, d.chunk_size, t, d.entries)
t2 = time.perf_counter()
print(json.dumps({"events": len(ev), "decompose_s": t1 - t0, "simulate_s": t2 - t1,
                  "violations": len(rep["violations"]), "kinds": sorted({v[0] for v in rep["violations"]}),
                  "completion_epoch": sched.completion_epoch, "sim_completion": rep["completion_epoch"],
                  "transfer_time_s": sched.transfer_time, "solve_device_s": sol.meta["device_seconds"]}))
