"""The CPU oracle against fixtures produced by the reference itself (CPU)."""

import numpy as np
import pytest

from oracle import lp_oracle
from tests.conftest import load_golden
from tests.golden.cases import CASES, build

MATRIX_KEYS = ("row_ptr", "col", "val", "row_lo", "row_hi", "var_lb", "var_ub", "obj")


@pytest.mark.parametrize("name", CASES)
def test_oracle_matrix_bit_exact(name):
    meta, gold = load_golden(name)
    t, d, tau, K, blim = build(name)
    a = lp_oracle.build_lp_arrays(t, d, tau, K, d.chunk_size, blim)
    for k in MATRIX_KEYS:
        assert a[k].dtype == gold[k].dtype or k in ("col",), k
        assert np.array_equal(a[k], gold[k]), k
    assert len(a["var_lb"]) == meta["num_vars"]
    assert len(a["row_lo"]) == meta["num_rows"]


@pytest.mark.parametrize("name", [c for c in CASES if c != "ndv2x2_ag1_K24"])
def test_oracle_highs_matches_reference(name):
    meta, gold = load_golden(name)
    t, d, tau, K, blim = build(name)
    a = lp_oracle.build_lp_arrays(t, d, tau, K, d.chunk_size, blim)
    res = lp_oracle.solve_highs(a, time_limit=60)
    assert res["status"] == meta["status"]
    if meta["status"] == "optimal":
        assert res["objective"] == pytest.approx(meta["objective"], rel=1e-9)
        assert lp_oracle.completion_epoch(a, res["x"]) == meta["completion_epoch"]
        viol = lp_oracle.replay_check(t, a, res["x"], tau, d.chunk_size)
        assert viol == {"capacity": 0, "causality": 0, "switch": 0, "unmet": 0}


def test_replay_flags_corruption():
    name = "dgx1_ag1_K8"
    meta, gold = load_golden(name)
    t, d, tau, K, blim = build(name)
    a = lp_oracle.build_lp_arrays(t, d, tau, K, d.chunk_size, blim)
    x = gold["x"].copy()
    # drop every flow: demand can no longer be met and reads lack backing
    for key, idx in a["columns"].items():
        if key[0] == "F":
            x[idx] = 0.0
    viol = lp_oracle.replay_check(t, a, x, tau, d.chunk_size)
    assert viol["causality"] > 0
