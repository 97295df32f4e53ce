import sys, os
sys.path.insert(0, os.getcwd())
from bench import workload
from paper_2305_13479_b200 import make_plan
from paper_2305_13479_b200.lp import build_from_plan
t, d, cfg = workload()
lp = build_from_plan(make_plan(t, d, cfg))
for mf in (0, 2, 3, 4):
    for cp in (0, 1):
        r = min((lp.step_bench(300, {"matrix_free": mf, "col_pipeline": cp}) for _ in range(3)), key=lambda r: r["ms_col"] + r["ms_row"])
        print(mf, cp, round(r["ms_col"] * 1e3, 2), round(r["ms_row"] * 1e3, 2), flush=True)
