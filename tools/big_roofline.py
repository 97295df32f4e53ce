"""Per-launch time and algorithmic-byte bandwidth of the iteration kernels on
LPs far larger than L2 (HBM-resident), for each operator: stored SELL matrix
(matrix_free 0), matrix-free per-entry (2) and segment (3) kernels.
usage: python tools/big_roofline.py [CHASSIS:K ...]   (default 8:1800 16:3860)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import peaks  # noqa: E402
from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand, make_plan  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

peak, kind = peaks()
specs = sys.argv[1:] or ["8:1800", "16:3860"]
# MODES: JSON list of matrix_free values or teccl_pdlp_opts override dicts
modes = [m if isinstance(m, dict) else {"matrix_free": m}
         for m in json.loads(os.environ.get("MODES", "[0, 2, 3, 4]"))]
for spec in specs:
    ch, K = (int(v) for v in spec.split(":"))
    t = ndv2(ch)
    d = generate_demand("allgather", t, 1, 25000)
    cfg = EpochConfig(epoch_duration(t, 25000, "fastest", 1), K, "fastest", 1, 25000)
    lp = build_from_plan(make_plan(t, d, cfg))
    reps = max(5, min(200, int(2e8 // lp.num_vars)))
    for mf in modes:
        best = None
        for _ in range(2):
            sb = lp.step_bench(reps, mf)
            if best is None or sb["ms_col"] + sb["ms_row"] < best["ms_col"] + best["ms_row"]:
                best = sb
        gc = best["bytes_col"] / (best["ms_col"] * 1e-3) / 1e9
        gr = best["bytes_row"] / (best["ms_row"] * 1e-3) / 1e9
        print(json.dumps({"chassis": ch, "K": K, "cols": lp.num_vars, "rows": lp.num_rows, "nnz": lp.nnz,
                          "opts": mf, "operator": best["matrix_free"], "ms_col": round(best["ms_col"], 4), "ms_row": round(best["ms_row"], 4),
                          "ms_iter": round(best["ms_col"] + best["ms_row"], 4),
                          "bytes_col": best["bytes_col"], "bytes_row": best["bytes_row"],
                          "gbs_col": round(gc, 1), "gbs_row": round(gr, 1),
                          "frac_col": round(gc / peak, 3), "frac_row": round(gr / peak, 3), "peak": peak}),
              flush=True)
    lp.close()
