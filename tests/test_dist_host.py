"""Host-side logic of the row-partitioned solve (CPU only): epoch-major
column map and epoch split."""

import numpy as np
import pytest

from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand, make_plan
from paper_2305_13479_b200.dist import em_to_ref_cols, partition_epochs
from paper_2305_13479_b200.topology import dgx2, ndv2


def _plan(t, kind, ch, K):
    d = generate_demand(kind, t, ch, 25000)
    return make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), K, "fastest", 1, 25000))


def test_em_column_map_is_a_permutation():
    for plan in (_plan(ndv2(2), "allgather", 1, 7), _plan(dgx2(1), "alltoall", 1, 5)):
        S, E, G, P, K = plan.S, plan.E, plan.G, plan.P, plan.K
        cw = S * E + S * G + 2 * P
        total = K * cw + S * G
        assert total == plan.num_vars
        ref = em_to_ref_cols(plan, 0, total)
        assert np.array_equal(np.sort(ref), np.arange(total))
        # epoch k's flows of source s, edge e sit at k*cw + s*E + e
        assert ref[3 * cw + 1 * E + 2] == plan.var_F(1, 2, 3)
        assert ref[K * cw + 0] == plan.var_B(0, 0, K)
        assert ref[2 * cw + S * E + S * G + 1] == plan.var_Rc(0, 2)


def test_partition_epochs_cover_horizon():
    for K, W in ((530, 2), (530, 8), (12, 3)):
        parts = partition_epochs(K, W)
        assert parts[0][0] == 0 and parts[-1][1] == K
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def test_solve_distributed_scheme_choice(monkeypatch):
    # auto: source partition while the LP fits the 31-bit single-device
    # indices, epoch blocks beyond; explicit schemes pass through
    from paper_2305_13479_b200 import dist as D
    calls = []
    monkeypatch.setattr(D, "solve_source_partitioned", lambda *a, **k: calls.append("source") or {})
    monkeypatch.setattr(D, "solve_partitioned", lambda *a, **k: calls.append("epoch") or {})
    t = ndv2(2)
    d = generate_demand("allgather", t, 1, 25000)
    cfg = EpochConfig(epoch_duration(t, 25000, "fastest", 1), 64, "fastest", 1, 25000)
    D.solve_distributed(t, d, cfg)
    D.solve_distributed(t, d, cfg, scheme="epoch")
    D.solve_distributed(t, d, cfg, scheme="source")
    assert calls == ["source", "epoch", "source"]
    with pytest.raises(ValueError):
        D.solve_distributed(t, d, cfg, scheme="nope")
