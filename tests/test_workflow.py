"""synthesize(t, d, method="lp") -- the reference's end-to-end LP workflow
(pkg/src/collsched/workflow.py:37-113) on the GPU engine."""

import pytest

from paper_2305_13479_b200 import ValidationError, generate_demand, synthesize
from paper_2305_13479_b200.lp import HYPER_EDGE
from paper_2305_13479_b200.topology import dgx1


def test_methods_outside_the_lp_path_are_refused():
    t = dgx1()
    d = generate_demand("allgather", t, 1, 25000)
    for m in ("milp", "astar", "nope"):
        with pytest.raises(ValidationError):
            synthesize(t, d, method=m, epochs=8)
    with pytest.raises(ValidationError):
        synthesize(t, d, switch_mode=HYPER_EDGE, epochs=8)


@pytest.mark.gpu
def test_synthesize_dgx1_alltoall_minimal_horizon():
    # reference acceptance instance: DGX1 AllToAll, 1 chunk, fastest-link
    # epochs -> minimal horizon 8 (tests/test_gpu_parity.py), schedule replays
    from oracle.simulator import simulate
    t = dgx1()
    d = generate_demand("alltoall", t, 1, 25000)
    r = synthesize(t, d, "lp", search_horizon=True, eps_rel=1e-6)
    assert r.epochs == 8 and r.report.ok
    assert r.schedule.completion_epoch == r.report.completion_epoch <= 7 and r.check.ok
    ev = [(e.source, e.chunk, e.src, e.dst, e.epoch, e.fraction) for e in r.schedule.events]
    rep = simulate(ev, r.tau, d.chunk_size, t, d.entries)
    assert rep["violations"] == [] and rep["completion_epoch"] == r.schedule.completion_epoch


@pytest.mark.gpu
def test_synthesize_without_horizon_uses_doubling_search():
    # K = 8 is the first doubling probe; the event replay (native simulate)
    # and the flow checker both pass before the schedule is returned
    t = dgx1()
    d = generate_demand("allgather", t, 1, 25000)
    r = synthesize(t, d)
    assert r.epochs == 8 and r.report.ok and r.check.ok and r.status == "optimal"
    assert any("doubling search" in w for w in r.warnings)
    assert r.report.completion_epoch <= r.schedule.completion_epoch
