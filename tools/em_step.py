"""Half-step kernels of one epoch-major block holding the whole LP (world 1):
stored SELL (matrix_free 0) vs the epoch-major matrix-free operator (2).
usage: python tools/em_step.py [CHASSIS:K ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand, make_plan  # noqa: E402
from paper_2305_13479_b200.dist import build_partition  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

for spec in sys.argv[1:] or ["8:1800"]:
    ch, K = (int(v) for v in spec.split(":"))
    t = ndv2(ch)
    d = generate_demand("allgather", t, 1, 25000)
    plan = make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), K, "fastest", 1, 25000))
    part = build_partition(plan, 1, 0)
    for mf in (0, 2):
        r = min((part.step_bench(20, {"matrix_free": mf}) for _ in range(2)), key=lambda r: r["ms_col"] + r["ms_row"])
        print(json.dumps({"chassis": ch, "K": K, "matrix_free": mf, "ms_col": round(r["ms_col"], 4),
                          "ms_row": round(r["ms_row"], 4),
                          "gbs_col": round(r["bytes_col"] / r["ms_col"] / 1e6, 1),
                          "gbs_row": round(r["bytes_row"] / r["ms_row"] / 1e6, 1)}), flush=True)
    part.close()
