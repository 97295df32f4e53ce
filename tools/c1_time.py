"""configs[1] to the parity bar, three solves: iterations, device seconds,
µs per iteration (L2 flushed before each)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
pdlp = json.loads(os.environ.get("PDLP_OPTS", "{}"))
for _ in range(4):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    sol = solve(lp, SolverOptions(pdlp=pdlp))
    print(json.dumps({"lib": os.environ.get("TECCL_B200_LIB", "default"), "iters": sol.meta["iters"],
                      "s": sol.meta["device_seconds"], "us_per_iter": 1e6 * sol.meta["device_seconds"] / sol.meta["iters"],
                      "objective": sol.objective}), flush=True)
