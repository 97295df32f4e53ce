"""Generate golden LP fixtures by running the REFERENCE package itself.

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py
For every case in cases.py it builds the model with collsched.lp.build_lp_model,
solves it with collsched.solver.solve (scipy HiGHS), and stores the canonical
CSR (columns ascending per row), bounds, minimisation costs, the reference's
status/objective/completion epoch and the optimal x, one .npz per case, plus
golden.json with the scalar results.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")

import collsched.demand as rdem  # noqa: E402
import collsched.epochs as rep  # noqa: E402
import collsched.topology as rtopo  # noqa: E402
from collsched.epochs import EpochConfig  # noqa: E402
from collsched.lp import build_lp_model, lp_completion_epoch, lp_rates_to_schedule  # noqa: E402
from collsched.milp import ModelOptions  # noqa: E402
from collsched.model import INF  # noqa: E402
from collsched.solver import SolverOptions, solve  # noqa: E402

from tests.golden.cases import CASES, build  # noqa: E402


def canonical(m):
    rows = []
    lo, hi = [], []
    for coeffs, rlo, rhi in m.rows:
        rows.append(sorted(coeffs))
        lo.append(-np.inf if rlo == -INF else rlo)
        hi.append(np.inf if rhi == INF else rhi)
    rp = np.zeros(len(rows) + 1, np.int64)
    for r, cf in enumerate(rows):
        rp[r + 1] = rp[r] + len(cf)
    c = np.zeros(m.num_vars)
    for idx, coef in m.objective.items():
        c[idx] = -coef
    return {
        "row_ptr": rp,
        "col": np.array([i for cf in rows for i, _ in cf], np.int32),
        "val": np.array([v for cf in rows for _, v in cf], np.float64),
        "row_lo": np.array(lo), "row_hi": np.array(hi),
        "var_lb": np.array(m.lb, np.float64),
        "var_ub": np.array([np.inf if b == INF else b for b in m.ub], np.float64),
        "obj": c,
    }


def main():
    ref_mod = {"topo": rtopo, "dem": rdem, "ep": rep}
    summary = {}
    for name in CASES:
        t_ref, d_ref, tau, K, blim = build(name, ref_mod)
        t_me, d_me, tau_me, K_me, _ = build(name)
        assert tau == tau_me and K == K_me
        assert [(e.src, e.dst, e.capacity, e.alpha) for e in t_ref.edges] == \
               [(e.src, e.dst, e.capacity, e.alpha) for e in t_me.edges], name
        assert tuple(t_ref.nodes) == tuple(t_me.nodes) and set(t_ref.switches) == set(t_me.switches)
        assert d_ref.entries == d_me.entries
        cfg = EpochConfig(tau, K, "fastest", 1, d_ref.chunk_size)
        m = build_lp_model(t_ref, d_ref, cfg, ModelOptions(buffer_limit=blim))
        arrays = canonical(m)
        sol = solve(m, SolverOptions(time_limit=600))
        entry = {"status": sol.status, "objective": sol.objective, "num_vars": m.num_vars,
                 "num_rows": len(m.rows), "nnz": int(arrays["row_ptr"][-1]), "K": K, "tau": tau,
                 "buffer_limit": blim}
        x = np.zeros(0)
        if sol.feasible:
            entry["completion_epoch"] = lp_completion_epoch(sol)
            x = np.asarray(sol.x)
            sched = lp_rates_to_schedule(sol, t_ref, d_ref, cfg)
            entry["schedule"] = [[e.source, e.chunk, e.src, e.dst, e.epoch, e.fraction]
                                 for e in sched.events]
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), x=x, **arrays)
        summary[name] = entry
        print(name, entry, flush=True)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
