import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
import ctypes as C
from bench import workload
from paper_2305_13479_b200 import SolverOptions, make_plan, solve
from paper_2305_13479_b200 import schedule as S
from paper_2305_13479_b200 import _native as nat
from paper_2305_13479_b200.lp import build_from_plan
t, d, cfg = workload(); plan = make_plan(t, d, cfg); lp = build_from_plan(plan)
sol = solve(lp, SolverOptions(eps_rel=1e-8))
x = S.repair_flows(plan, np.asarray(sol.x))
lib = nat.load()
orig = lib.teccl_schedule_te
tm = {}
def wrapped(*a):
    t0 = time.perf_counter(); r = orig(*a); tm["c_schedule_te"] = time.perf_counter() - t0; return r
lib.teccl_schedule_te = wrapped
t0 = time.perf_counter(); ev = S.decompose_native(plan, x, S.DUST); tm["total"] = time.perf_counter() - t0
for th in (1, 4, 16, 32):
    lib.teccl_schedule_te = orig
    t0 = time.perf_counter(); S.decompose_native(plan, x, S.DUST, threads=th); tm[f"total_threads{th}"] = time.perf_counter() - t0
print(json.dumps(tm), os.cpu_count())
