"""Smallest feasible horizon of the configs[1] LP, by phase-1 solves on the GPU."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import make_plan  # noqa: E402
from paper_2305_13479_b200.lp import feasibility_gap  # noqa: E402

t, d, cfg = workload()
out = {}
for K in [int(v) for v in sys.argv[1].split(",")]:
    t0 = time.perf_counter()
    gap = feasibility_gap(make_plan(t, d, cfg.with_horizon(K)))
    out[K] = {"unmet_chunks": gap, "seconds": time.perf_counter() - t0}
    print(K, out[K], flush=True)
print(json.dumps(out))
