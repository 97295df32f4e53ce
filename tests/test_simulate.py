"""Native event replay (csrc/simulate.cu via simulate.py) against the
reference's own simulate() outputs (tests/golden/sim_golden.json, made by
make_golden_sim.py from collsched/simulator.py:58-208): every violation in
order, per-entry and per-destination completion, transfer time. Host code
only -- runs without a GPU."""

import json
import os

import pytest

from paper_2305_13479_b200.errors import ScheduleError, ValidationError
from paper_2305_13479_b200.schedule import Schedule, ScheduleEvent
from paper_2305_13479_b200.simulate import SimOptions, algorithmic_bandwidth, simulate
from tests.golden.cases import build

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "sim_golden.json")))


def _key(v):
    return tuple(v) if isinstance(v, list) else v


@pytest.mark.parametrize("name", sorted(GOLD))
def test_native_replay_matches_reference(name):
    g = GOLD[name]
    t, d, tau, K, _ = build(g["case"])
    sched = Schedule(tau=tau, events=tuple(ScheduleEvent(*e) for e in g["events"]),
                     completion_epoch=-1, chunk_size=d.chunk_size)
    rpt = simulate(sched, t, d, SimOptions(switch_mode=g["switch_mode"]))
    got = [[v.kind, v.location, v.epoch] for v in rpt.violations]
    assert got == g["violations"]
    assert rpt.completion_epoch == g["completion_epoch"]
    assert rpt.transfer_time == g["transfer_time"]
    assert {(s, c, dst): k for s, c, dst, k in g["per_entry"]} == rpt.per_entry_completion
    assert {dst: k for dst, k in g["completion_epochs"]} == rpt.completion_epochs


@pytest.mark.parametrize("name", [n for n in sorted(GOLD) if GOLD[n]["switch_mode"] == "copy"])
def test_oracle_replay_matches_reference(name):
    # pins the test-only restatement (oracle/simulator.py) to the same fixtures
    from oracle.simulator import simulate as oracle_simulate
    g = GOLD[name]
    t, d, tau, K, _ = build(g["case"])
    r = oracle_simulate([tuple(e) for e in g["events"]], tau, d.chunk_size, t, d.entries)
    assert [list(v) for v in r["violations"]] == g["violations"]
    assert r["completion_epoch"] == g["completion_epoch"]


def test_replay_input_errors_match_reference_messages():
    t, d, tau, K, _ = build("dgx1_ag1_K8")
    ok = GOLD["dgx1_ag1_K8/as_emitted"]["events"]
    bad_edge = [list(e) for e in ok] + [[0, 0, 0, 99, 1, 0.5]]
    with pytest.raises(ScheduleError, match=r"unknown edge \(0,99\)"):
        simulate(Schedule(tau, tuple(ScheduleEvent(*e) for e in bad_edge), -1, d.chunk_size), t, d)
    e0 = list(ok[0])
    e0[5] = 1.5
    with pytest.raises(ScheduleError, match="outside"):
        simulate(Schedule(tau, (ScheduleEvent(*e0),), -1, d.chunk_size), t, d)
    with pytest.raises(ValidationError):
        simulate(Schedule(tau, (), -1, d.chunk_size), t, d, SimOptions(switch_mode="hyper-edge"))
    with pytest.raises(ScheduleError, match="not a node"):
        simulate(Schedule(tau, (ScheduleEvent("nope", 0, 0, 1, 0, 1.0),), -1, d.chunk_size), t, d)


def test_empty_schedule_reports_every_entry_unmet():
    t, d, tau, K, _ = build("star3_K5")
    rpt = simulate(Schedule(tau, (), -1, d.chunk_size), t, d)
    assert [v.kind for v in rpt.violations] == ["unmet-demand"] * len(d.entries)
    assert rpt.completion_epoch == -1 and rpt.transfer_time == 0.0


def test_algorithmic_bandwidth():
    g = GOLD["dgx1_ag1_K8/as_emitted"]
    t, d, tau, K, _ = build("dgx1_ag1_K8")
    rpt = simulate(Schedule(tau, tuple(ScheduleEvent(*e) for e in g["events"]), -1, d.chunk_size), t, d)
    bw = algorithmic_bandwidth(rpt)
    assert bw["aggregate"] == pytest.approx(sum(rpt.output_buffer_bytes.values()) / rpt.transfer_time)
