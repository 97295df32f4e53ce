"""Solve statuses as the reference reports them (collsched/solver.py:128-168):
"infeasible" from the device's Farkas certificate, "optimal" only at
north_star's parity bar (duality gap <= 1e-4 AND relative primal / dual
residuals <= 1e-6), and the reference's own min_feasible_horizon loop driven
through the INTEGRATION.md hook."""

import types

import numpy as np
import pytest

from paper_2305_13479_b200 import (EpochConfig, ModelOptions, SolverOptions, build_lp_model,
                                   make_plan, solve)
from paper_2305_13479_b200.errors import HorizonInfeasibleError, SolverBackendError
from paper_2305_13479_b200.hook import reference_solve
from paper_2305_13479_b200.lp import build_from_plan
from tests.conftest import load_golden
from tests.golden.cases import CASES, build

pytestmark = pytest.mark.gpu

INFEASIBLE_CASES = ["dgx1_ag1_K6", "ndv2x2_ag1_K24"]
OPTIMAL_CASES = [c for c in CASES if c not in INFEASIBLE_CASES]


def _model(name):
    t, d, tau, K, blim = build(name)
    return build_lp_model(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size),
                          ModelOptions(buffer_limit=blim))


@pytest.mark.parametrize("name", INFEASIBLE_CASES)
def test_infeasible_goldens_are_certified(name):
    meta, _ = load_golden(name)
    assert meta["status"] == "infeasible"
    sol = solve(_model(name), SolverOptions(max_iters=200_000, time_limit=60))
    assert sol.status == "infeasible", sol.meta
    assert sol.x is None and sol.objective is None          # like the reference's Solution
    assert sol.meta["infeas_cert"] > 1e-6
    assert sol.meta["iters"] < 200_000


@pytest.mark.parametrize("name", OPTIMAL_CASES)
def test_parity_bar_default_solve(name):
    # the default solve stops at the parity bar and matches the reference's optimum
    meta, _ = load_golden(name)
    sol = solve(_model(name), SolverOptions(time_limit=120))
    assert sol.status == "optimal", sol.meta
    assert sol.meta["rel_gap"] <= 1e-4
    assert sol.meta["rel_primal_res"] <= 1e-6 and sol.meta["rel_dual_res"] <= 1e-6
    assert sol.objective == pytest.approx(meta["objective"], rel=1e-4, abs=1e-6)


def test_iteration_cap_is_timeout():
    sol = solve(_model("dgx1_ag1_K6"), SolverOptions(max_iters=64, eps_infeas=0.0))
    assert sol.status == "timeout" and sol.x is not None


def _reference_style_model(t, d, cfg, opts=None):
    """Stand-in for a collsched Model from build_lp_model (lp.py:40-45): the
    meta it records plus its size (the reference package is not on the GPU
    box; the device rebuild is pinned to it by the builder goldens)."""
    plan = make_plan(t, d, cfg, opts)
    return types.SimpleNamespace(
        meta={"kind": "lp", "topology": t, "demand": d, "cfg": cfg, "opts": opts},
        num_vars=plan.num_vars, rows=[None] * plan.num_rows, kinds=["C"] * plan.num_vars)


def _reference_min_feasible_horizon(builder, k_lo, k_hi, opts, solve_fn):
    """collsched.solver.min_feasible_horizon, statement for statement
    (solver.py:146-168), with `solve` = the backend hook."""
    best = None
    lo, hi = k_lo, k_hi
    while lo <= hi:
        mid = (lo + hi) // 2
        sol = solve_fn(builder(mid), opts)
        if sol.status == "timeout":
            raise SolverBackendError(f"horizon probe timed out at K={mid}")
        if sol.feasible:
            best = (mid, sol)
            hi = mid - 1
        else:
            lo = mid + 1
    if best is None:
        raise HorizonInfeasibleError(k_lo, k_hi)
    return best


def test_reference_horizon_search_through_hook():
    from paper_2305_13479_b200 import epoch_duration, generate_demand
    from paper_2305_13479_b200.topology import dgx1
    t = dgx1()
    d = generate_demand("allgather", t, 1, 25000)
    tau = epoch_duration(t, 25000, "fastest", 1)
    builder = lambda k: _reference_style_model(t, d, EpochConfig(tau, k, "fastest", 1, 25000))
    opts = types.SimpleNamespace(time_limit=60.0, verbosity=0)
    k, sol = _reference_min_feasible_horizon(builder, 1, 12, opts, reference_solve)
    assert k == 8
    meta, gold = load_golden("dgx1_ag1_K8")
    assert sol.objective == pytest.approx(meta["objective"], rel=1e-4)
    assert len(sol.x) == len(gold["var_lb"])


def test_min_feasible_horizon_frees_probes_and_raises_on_timeout():
    from paper_2305_13479_b200 import min_feasible_horizon
    t, d, tau, K, _ = build("dgx1_ag1_K8")
    built = []

    def builder(k):
        lp = build_lp_model(t, d, EpochConfig(tau, k, "fastest", 1, d.chunk_size))
        built.append(lp)
        return lp
    k, sol = min_feasible_horizon(builder, 1, 12, SolverOptions())
    assert k == 8
    assert all(lp.handle is None for lp in built if lp is not sol.model)  # discarded probes freed
    with pytest.raises(SolverBackendError, match="timed out"):
        min_feasible_horizon(builder, 1, 12, SolverOptions(max_iters=64))


def test_phase1_probe_raises_when_not_converged():
    from paper_2305_13479_b200.lp import feasibility_gap
    t, d, tau, K, _ = build("dgx1_ag1_K8")
    with pytest.raises(SolverBackendError, match="phase-1"):
        feasibility_gap(make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size)), max_iters=64)


def test_certificate_off_for_feasible_lp_family():
    # every feasible configs[0]-family horizon solves to optimal: the
    # certificate never fires on a feasible LP (it cannot, up to rounding)
    from paper_2305_13479_b200 import epoch_duration, generate_demand
    from paper_2305_13479_b200.topology import dgx1
    t = dgx1()
    d = generate_demand("allgather", t, 1, 25000)
    tau = epoch_duration(t, 25000, "fastest", 1)
    for K in (8, 9, 16, 40):
        lp = build_from_plan(make_plan(t, d, EpochConfig(tau, K, "fastest", 1, 25000)))
        sol = solve(lp, SolverOptions(eps_infeas=1e-12))
        assert sol.status == "optimal", (K, sol.meta)
        assert np.isfinite(sol.objective)
        lp.close()


def _golden_model(name, with_meta=True):
    """A collsched Model as the hook receives it: the reference's own rows,
    bounds and objective (the golden .npz is collsched's build_lp_model
    output) and, like every Model build_lp_model makes, meta kind "lp" with
    the inputs it was built from (lp.py:40-45)."""
    meta_g, a = load_golden(name)
    t, d, tau, K, blim = build(name)
    rp, col, val = a["row_ptr"], a["col"], a["val"]
    rows = [(list(zip(col[rp[r]:rp[r + 1]].tolist(), val[rp[r]:rp[r + 1]].tolist())),
             a["row_lo"][r], a["row_hi"][r]) for r in range(len(rp) - 1)]
    meta = {"kind": "lp", "topology": t, "demand": d,
            "cfg": EpochConfig(tau, K, "fastest", 1, d.chunk_size),
            "opts": ModelOptions(buffer_limit=blim)} if with_meta else {}
    return meta_g, types.SimpleNamespace(
        name="lp-alltoall", num_vars=len(a["var_lb"]), kinds=["C"] * len(a["var_lb"]),
        lb=list(a["var_lb"]), ub=list(a["var_ub"]), rows=rows,
        objective={j: -c for j, c in enumerate(a["obj"]) if c}, meta=meta)


@pytest.mark.parametrize("name", ["dgx1_ag1_K8", "dgx1_ag1_K6", "ndv2x2_ag1_K24", "funnel_blimit_K4"])
def test_hook_on_reference_model_data(name):
    # through the hook with the reference's own model data: the status and
    # objective the reference's HiGHS reported (golden.json)
    meta_g, m = _golden_model(name)
    sol = reference_solve(m, types.SimpleNamespace(time_limit=60.0, verbosity=0))
    assert sol.status == meta_g["status"]
    if sol.feasible:
        assert sol.objective == pytest.approx(meta_g["objective"], rel=1e-4)
        assert len(sol.x) == m.num_vars


def test_hook_generic_upload_without_meta():
    # a Model without build_lp_model's meta goes through the CSR upload
    meta_g, m = _golden_model("dgx1_ag1_K8", with_meta=False)
    sol = reference_solve(m, types.SimpleNamespace(time_limit=60.0, verbosity=0))
    assert sol.status == "optimal"
    assert sol.objective == pytest.approx(meta_g["objective"], rel=1e-4)
