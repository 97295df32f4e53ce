"""A/B of iteration-kernel variants on configs[1]: matrix-free operator vs
stored SELL matrix, programmatic dependent launch on/off, pipelined column
kernel. Prints iterations, device seconds and us/iteration per variant."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import SolverOptions, make_plan, solve  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402

t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
variants = [dict(matrix_free=mf, pdl=pdl, col_pipeline=cp)
            for mf, pdl, cp in itertools.product((3, 2, 0), (1, 0), (1,))]
variants.append(dict(matrix_free=0, pdl=1, col_pipeline=0))
if os.environ.get("VARIANTS"):  # e.g. '[{"matrix_free": 0, "pdl": 1, "col_pipeline": 1}]'
    import json
    variants = json.loads(os.environ["VARIANTS"])
for v in variants:
    opts = SolverOptions(eps_rel=1e-4, pdlp=v)
    best = None
    for _ in range(3):
        s = solve(lp, opts)
        if best is None or s.meta["device_seconds"] < best.meta["device_seconds"]:
            best = s
    sb = lp.step_bench(100) if v["pdl"] == 1 else None
    print(os.path.basename(os.environ.get("TECCL_B200_LIB", "default")), v, best.meta["iters"], round(best.meta["device_seconds"], 4),
          round(1e6 * best.meta["device_seconds"] / best.meta["iters"], 2), "us/it",
          round(best.objective, 6), flush=True)
