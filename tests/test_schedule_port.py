"""Rate -> schedule decomposition against the reference's own schedules
(CPU): the port applied to the reference's HiGHS solution must reproduce
collsched.lp_rates_to_schedule's event list exactly."""

import pytest

from paper_2305_13479_b200 import EpochConfig, make_plan
from paper_2305_13479_b200.errors import ConservationError
from paper_2305_13479_b200.lp import ModelOptions
from paper_2305_13479_b200.schedule import decompose
from tests.conftest import load_golden
from tests.golden.cases import CASES, build

SCHEDULED = [c for c in CASES if c not in ("dgx1_ag1_K6", "ndv2x2_ag1_K24")]


def _plan(name):
    t, d, tau, K, blim = build(name)
    return make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size), ModelOptions(buffer_limit=blim))


@pytest.mark.parametrize("name", SCHEDULED)
def test_decomposition_matches_reference_exactly(name):
    meta, gold = load_golden(name)
    events = decompose(_plan(name), gold["x"])
    got = [[e.source, e.chunk, e.src, e.dst, e.epoch, e.fraction] for e in events]
    assert got == meta["schedule"]


def test_parallel_paths_split_in_halves():
    # reference test_lp.py:82-97: two 0.5 paths carry one chunk
    meta, gold = load_golden("parallel_K2")
    events = decompose(_plan("parallel_K2"), gold["x"])
    assert sorted(e.fraction for e in events) == pytest.approx([0.5] * 4)


def test_zero_rate_solution_raises():
    # reference test_lp.py:100-107
    meta, gold = load_golden("single_edge_K2")
    plan = _plan("single_edge_K2")
    x = gold["x"].copy()
    x[:plan.S * plan.SB] = 0.0
    for k in range(plan.K):
        x[plan.var_F(0, 0, k)] = 0.0
    with pytest.raises(ConservationError, match="residue|backing"):
        decompose(plan, x)


@pytest.mark.parametrize("name", SCHEDULED)
def test_reference_schedules_replay_clean(name):
    # the oracle's simulator restatement accepts the reference's own schedules
    from oracle.simulator import simulate
    meta, gold = load_golden(name)
    t, d, tau, K, blim = build(name)
    rep = simulate(meta["schedule"], tau, d.chunk_size, t, d.entries)
    assert rep["violations"] == []
    assert rep["completion_epoch"] == meta["completion_epoch"]


def test_oracle_simulator_flags_overload():
    from oracle.simulator import simulate
    meta, gold = load_golden("single_edge_K2")
    t, d, tau, K, blim = build("single_edge_K2")
    ev = [list(e) for e in meta["schedule"]] + [[0, 0, 0, 1, 0, 1.0]]
    rep = simulate(ev, tau, d.chunk_size, t, d.entries)
    assert any(v[0] == "capacity" for v in rep["violations"])


@pytest.mark.parametrize("name", SCHEDULED)
def test_vertex_solutions_need_no_repair(name):
    from paper_2305_13479_b200.schedule import RAW_OK, max_deficit
    meta, gold = load_golden(name)
    assert max_deficit(_plan(name), gold["x"]) <= RAW_OK


def test_repair_makes_perturbed_solution_decomposable():
    # perturb an exact solution the way a first-order solver leaves it (1e-7
    # imbalances); repair + decomposition must still serve every read
    import numpy as np
    from paper_2305_13479_b200.schedule import max_deficit, repair_flows
    meta, gold = load_golden("dgx1_ag1_K10")
    plan = _plan("dgx1_ag1_K10")
    rng = np.random.default_rng(0)
    x = gold["x"] * (1.0 + 1e-7 * rng.standard_normal(gold["x"].shape))
    assert max_deficit(plan, x) > 0
    y = repair_flows(plan, x)
    assert max_deficit(plan, y) <= 1e-12
    events = decompose(plan, y)
    from oracle.simulator import simulate
    t, d, tau, K, blim = build("dgx1_ag1_K10")
    rep = simulate([(e.source, e.chunk, e.src, e.dst, e.epoch, e.fraction) for e in events],
                   tau, d.chunk_size, t, d.entries)
    assert rep["violations"] == []


@pytest.mark.parametrize("name", SCHEDULED)
def test_native_decomposition_matches_reference_exactly(name):
    import os
    from paper_2305_13479_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libteccl_b200.so not built")
    from paper_2305_13479_b200.schedule import decompose_native
    meta, gold = load_golden(name)
    events = decompose_native(_plan(name), gold["x"])
    got = [[e.source, e.chunk, e.src, e.dst, e.epoch, e.fraction] for e in events]
    assert got == meta["schedule"]


def test_native_and_python_agree_after_repair():
    import numpy as np
    from paper_2305_13479_b200.schedule import DUST, decompose_native, repair_flows
    meta, gold = load_golden("dgx2x1_a2a_K20")
    plan = _plan("dgx2x1_a2a_K20")
    rng = np.random.default_rng(1)
    y = repair_flows(plan, gold["x"] * (1.0 + 1e-7 * rng.standard_normal(gold["x"].shape)))
    a = decompose(plan, y, DUST)
    b = decompose_native(plan, y, DUST)
    assert a == b
