"""configs[2]: ALLTOALL on the DGX-2 family (per-link alpha/beta: 125 GB/s
switch links with 0.35 us latency, 12.5 GB/s cross-chassis links with
2.6 us -- collsched.topology.dgx2, reference topology.py:276-299).

* 2-chassis AllToAll at its smallest feasible horizon K* = 333 against the
  reference's own optimum (tests/golden/full_size_dgx2.json: collsched's
  build_lp_model + HiGHS), and K* - 1 certified infeasible on the device.
* 4-chassis AllToAll (configs[2] itself, 43.3M columns) at K* = 1933: solved to
  1e-8 with its duality-gap certificate, finish epoch 1932 and a clean
  integer replay. (K = 1932 is certified infeasible in
  profiles/r02_c_config2_horizon.log -- 974k iterations, too long for a test.)
"""

import json
import os

import pytest

from paper_2305_13479_b200 import (EpochConfig, SolverOptions, build_lp_model, check_lp_schedule,
                                   epoch_duration, generate_demand, lp_completion_epoch, make_plan, solve)
from paper_2305_13479_b200.lp import build_from_plan
from paper_2305_13479_b200.topology import dgx2

pytestmark = pytest.mark.gpu
GOLD_PATH = os.path.join(os.path.dirname(__file__), "golden", "full_size_dgx2.json")


def _cfg(chassis, K):
    t = dgx2(chassis)
    d = generate_demand("alltoall", t, 1, 25000)
    tau = epoch_duration(t, 25000, "fastest", 1)
    return t, d, EpochConfig(tau, K, "fastest", 1, 25000)


def test_dgx2x2_alltoall_matches_reference_optimum():
    gold = json.load(open(GOLD_PATH))["dgx2x2_a2a1_K333"]
    t, d, cfg = _cfg(2, 333)
    lp = build_lp_model(t, d, cfg)
    assert (lp.num_vars, lp.num_rows) == (gold["num_vars"], gold["num_rows"])
    sol = solve(lp, SolverOptions(time_limit=120))          # parity bar
    assert sol.status == "optimal"
    assert sol.objective == pytest.approx(gold["objective"], rel=1e-4)
    assert sol.meta["rel_primal_res"] <= 1e-6 and sol.meta["rel_dual_res"] <= 1e-6
    assert lp_completion_epoch(sol, tol=1e-5) == gold["completion_epoch"]
    lp.close()


def test_dgx2x2_alltoall_one_epoch_short_is_infeasible():
    t, d, cfg = _cfg(2, 332)
    sol = solve(build_lp_model(t, d, cfg), SolverOptions(time_limit=300, max_iters=5_000_000))
    assert sol.status == "infeasible", sol.meta
    gold = json.load(open(GOLD_PATH)).get("dgx2x2_a2a1_K332")
    if gold is not None and gold.get("status") in (0, 2):
        assert gold["status"] == 2  # HiGHS: infeasible


def test_config2_four_chassis_certified_optimum():
    t, d, cfg = _cfg(4, 1933)
    plan = make_plan(t, d, cfg)
    lp = build_from_plan(plan)
    assert lp.num_vars == 43_303_296
    sol = solve(lp, SolverOptions(eps_rel=1e-8, time_limit=600, max_iters=5_000_000))
    assert sol.status == "optimal"
    # duality-gap certificate: primal and dual objectives agree to 1e-8
    p, dual = sol.objective, sol.meta["dual_objective"]
    assert abs(p - dual) <= 1e-8 * max(1.0, abs(p), abs(dual))
    assert sol.meta["rel_primal_res"] <= 1e-8 and sol.meta["rel_dual_res"] <= 1e-8
    assert p == pytest.approx(9007.0162, rel=1e-7)          # profiles/r02_c_config2_horizon.log
    assert lp_completion_epoch(sol, tol=1e-5) == 1932
    rep = check_lp_schedule(plan, sol.x, tol=1e-5)
    assert rep.ok and rep.completion_epoch == 1932
    lp.close()
