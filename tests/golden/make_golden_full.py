"""Full-size golden values for the benchmark LPs, from the REFERENCE package.

Builds the configs[1] LP (2-chassis NDv2 AllGather) with collsched.lp.build_lp_model
and solves it with HiGHS through scipy (interior point + crossover: the
reference's default simplex path, collsched.solver.solve, does not finish it
in 10 minutes on an 8-core host; the optimum is unique in value, so the
method does not change the golden objective). Writes full_size.json.
Takes ~25 minutes for K=530. Run in the build container:
    python tests/golden/make_golden_full.py
"""

import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from collsched import generate_demand  # noqa: E402
from collsched.epochs import EpochConfig, epoch_duration  # noqa: E402
from collsched.lp import build_lp_model, lp_completion_epoch  # noqa: E402
from collsched.milp import ModelOptions  # noqa: E402
from collsched.model import INF  # noqa: E402
from collsched.solver import OPTIMAL, Solution  # noqa: E402
from collsched.topology import ndv2  # noqa: E402

CASES = {"ndv2x2_ag2_K530": (2, 530), "ndv2x2_ag1_K270": (1, 270)}


def solve_ipm(m):
    n = m.num_vars
    c = np.zeros(n)
    for i, v in m.objective.items():
        c[i] = -v
    r, ci, val, lo, hi = [], [], [], [], []
    for ri, (coeffs, rlo, rhi) in enumerate(m.rows):
        for idx, coef in coeffs:
            r.append(ri); ci.append(idx); val.append(coef)
        lo.append(-np.inf if rlo == -INF else rlo)
        hi.append(np.inf if rhi == INF else rhi)
    A = sp.csr_matrix((val, (r, ci)), shape=(len(m.rows), n))
    lo, hi = np.array(lo), np.array(hi)
    eq = lo == hi
    le = (~eq) & np.isfinite(hi)
    ge = (~eq) & np.isfinite(lo)
    ub = np.array([np.inf if b == INF else b for b in m.ub])
    t0 = time.time()
    res = linprog(c, A_ub=sp.vstack([A[le], -A[ge]]), b_ub=np.concatenate([hi[le], -lo[ge]]),
                  A_eq=A[eq], b_eq=lo[eq], bounds=np.stack([np.array(m.lb), ub], 1),
                  method="highs-ipm", options={"time_limit": 20000})
    return res, time.time() - t0


def main():
    out = {}
    for name, (ch, K) in CASES.items():
        t = ndv2(2)
        d = generate_demand("allgather", t, ch, 25000)
        tau = epoch_duration(t, d.chunk_size, "fastest", 1)
        m = build_lp_model(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size), ModelOptions())
        res, secs = solve_ipm(m)
        sol = Solution(OPTIMAL, m, np.asarray(res.x), float(-res.fun))
        out[name] = {"chunks": ch, "K": K, "objective": float(-res.fun),
                     "completion_epoch": lp_completion_epoch(sol), "highs_ipm_seconds": secs,
                     "num_vars": m.num_vars, "num_rows": len(m.rows)}
        print(name, out[name], flush=True)
    with open(os.path.join(HERE, "full_size.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
