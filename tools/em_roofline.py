"""Stored-SELL iteration kernels on the epoch-major numbering (the partition
builder at world = 1) vs the reference numbering, on LPs larger than L2.
usage: python tools/em_roofline.py [CHASSIS:K ...]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import _native as nat  # noqa: E402
from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand, make_plan  # noqa: E402
from paper_2305_13479_b200.dist import build_partition  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402


def sb(ctx, h, reps):
    out = (C.c_double * 6)()
    nat.check(ctx.lib.teccl_pdlp_step_bench(ctx.handle, h, int(reps), out))
    return out[0], out[1], out[2], out[3]


for spec in sys.argv[1:] or ["8:1800", "16:3860"]:
    ch, K = (int(v) for v in spec.split(":"))
    t = ndv2(ch)
    d = generate_demand("allgather", t, 1, 25000)
    cfg = EpochConfig(epoch_duration(t, 25000, "fastest", 1), K, "fastest", 1, 25000)
    plan = make_plan(t, d, cfg)
    reps = max(5, min(200, int(2e8 // plan.num_vars)))
    for name in ("reference", "epoch-major"):
        if name == "reference":
            lp = build_from_plan(plan)
            ctx, h = lp.ctx, lp.handle
        else:
            lp = build_partition(plan, 1, 0)
            ctx, h = lp.ctx, lp.handle
        best = min((sb(ctx, h, reps) for _ in range(2)), key=lambda r: r[0] + r[1])
        print(json.dumps({"chassis": ch, "K": K, "numbering": name, "ms_col": round(best[0], 4),
                          "ms_row": round(best[1], 4), "ms_iter": round(best[0] + best[1], 4),
                          "gbs_col": round(best[2] / best[0] / 1e6, 1),
                          "gbs_row": round(best[3] / best[1] / 1e6, 1)}), flush=True)
        lp.close()
