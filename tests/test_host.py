"""Host-side mirror of the reference's data formats (CPU only)."""

import json

import numpy as np
import pytest

from paper_2305_13479_b200 import (Demand, EpochConfig, ValidationError, compute_delta,
                                   epoch_duration, generate_demand, make_plan, merge_demands,
                                   validate_topology)
from paper_2305_13479_b200.lp import ModelOptions
from paper_2305_13479_b200.topology import (Edge, Topology, dgx1, dgx2, line, ndv2, ring, star,
                                            topology_from_json, topology_to_json)
from tests.conftest import load_golden
from tests.golden.cases import CASES, build


@pytest.mark.parametrize("name", CASES)
def test_plan_dimensions_match_reference(name):
    meta, gold = load_golden(name)
    t, d, tau, K, blim = build(name)
    plan = make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size), ModelOptions(buffer_limit=blim))
    assert plan.num_vars == meta["num_vars"]
    assert plan.num_rows == meta["num_rows"]
    # objective lives exactly on the Rc columns of the plan layout
    obj = gold["obj"]
    for p in range(plan.P):
        for k in range(K):
            assert obj[plan.var_Rc(p, k)] == -1.0 / (k + 1)
            assert obj[plan.var_Rd(p, k)] == 0.0
    # fixed Rc at the last epoch
    for p, (_, u) in enumerate(plan.pairs):
        assert gold["var_lb"][plan.var_Rc(p, K - 1)] == u


def test_capacities_bit_exact_with_reference_rows():
    meta, gold = load_golden("ndv2x2_ag1_K24")
    t, d, tau, K, blim = build("ndv2x2_ag1_K24")
    plan = make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size))
    S = plan.S
    cap_rows = gold["row_hi"][S:S + plan.E * K]
    assert np.array_equal(cap_rows, plan.cap)


def test_validate_topology_rules():
    assert validate_topology(star(3)) == []
    t = Topology(("a", "b"), frozenset(), (Edge("a", "b", 0.0),))
    assert len(validate_topology(t)) == 1
    t = Topology(("a", "b", "sw"), frozenset({"sw"}), (Edge("a", "sw", 1.0), Edge("a", "b", 1.0)))
    assert any("no outgoing edge" in v for v in validate_topology(t))


def test_generators_shapes():
    assert len(dgx1().edges) == 32
    t = ndv2(4)
    assert len(t.nodes) == 33 and len(t.edges) == 4 * 32 + 8
    t = dgx2(2)
    assert len(t.nodes) == 34
    assert len([e for e in t.edges if e.capacity == 12.5e9]) == 16
    assert len(ring(5).edges) == 10 and len(line(5).edges) == 8


def test_json_round_trip():
    t = ndv2(2)
    assert topology_from_json(json.loads(json.dumps(topology_to_json(t)))) == t


def test_demand_rules():
    d = generate_demand("allgather", dgx1(), 1, 25000)
    assert len(d.entries) == 56 and d.chunk_count == 8
    with pytest.raises(ValidationError):
        Demand(frozenset({(0, 0, 0)}), 1, 1)
    with pytest.raises(ValidationError):
        Demand(frozenset({(0, 0, 1), (1, 0, 2)}), 1, 1)
    a = generate_demand("allgather", line(2), 1, 8)
    b = generate_demand("alltoall", line(2), 1, 8)
    m = merge_demands([a, b])
    assert m.chunk_count == a.chunk_count + b.chunk_count
    with pytest.raises(ValidationError):
        merge_demands([a, generate_demand("allgather", line(2), 1, 16)])


def test_epoch_arithmetic():
    assert compute_delta(Edge("a", "b", 50e9, 0.7e-6), 0.5e-6) == 2
    assert compute_delta(Edge("a", "b", 1.0, 1.3e-6), 1.3e-6) == 1
    assert compute_delta(Edge("a", "b", 1.0, 0.0), 0.5) == 0
    assert epoch_duration(dgx1(), 25000, "fastest", 1) == pytest.approx(0.5e-6)
    assert epoch_duration(dgx1(), 25000, "slowest", 1) == pytest.approx(1.0e-6)
    with pytest.raises(ValidationError):
        EpochConfig(0.0, 4)


def test_plan_rejects_switch_endpoint():
    t = star(3)
    d = Demand(frozenset({("s", 0, "h")}), 1, 1)
    with pytest.raises(ValidationError):
        make_plan(t, d, EpochConfig(1.0, 2))
