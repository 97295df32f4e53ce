"""Golden replay fixtures for the native event simulator, made by running the
REFERENCE's own simulate() (collsched/simulator.py:58-208).

Run in the build container (needs /root/reference):
    python tests/golden/make_golden_sim.py
For every golden case with a schedule (golden.json, itself the reference's
lp_rates_to_schedule output) it replays the schedule as emitted and a few
deterministic corruptions -- a dropped delivery, a send moved one epoch
early, a doubled send, all fractions rounded up to whole chunks (windowed
capacity and widened delays), the no-copy switch mode -- and stores the
events with the reference's SimReport in sim_golden.json.
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")

import collsched.demand as rdem  # noqa: E402
import collsched.epochs as rep  # noqa: E402
import collsched.topology as rtopo  # noqa: E402
from collsched.schedule import Schedule, ScheduleEvent  # noqa: E402
from collsched.simulator import SimOptions, simulate  # noqa: E402

from tests.golden.cases import build  # noqa: E402


def variants(events, has_switch):
    """(name, events, switch_mode) -- deterministic corruptions."""
    out = [("as_emitted", events, "copy")]
    if not events:
        return out
    last = max(range(len(events)), key=lambda i: (events[i][4], i))
    out.append(("drop_last", events[:last] + events[last + 1:], "copy"))
    later = [i for i, e in enumerate(events) if e[4] > 0]
    if later:
        i = later[len(later) // 2]
        ev = list(events[i])
        ev[4] -= 1
        out.append(("early", events[:i] + [ev] + events[i + 1:], "copy"))
    i = len(events) // 3
    out.append(("doubled", events + [list(events[i])], "copy"))
    out.append(("whole", [e[:5] + [1.0] for e in events], "copy"))
    if has_switch:
        out.append(("no_copy", events, "no-copy"))
    return out


def main():
    ref_mod = {"topo": rtopo, "dem": rdem, "ep": rep}
    gold = json.load(open(os.path.join(HERE, "golden.json")))
    out = {}
    for name, g in sorted(gold.items()):
        if "schedule" not in g:
            continue
        t, d, tau, K, blim = build(name, ref_mod)
        for vname, evs, mode in variants([list(e) for e in g["schedule"]], bool(t.switches)):
            sched = Schedule(tau=tau, events=tuple(ScheduleEvent(*e) for e in evs),
                             completion_epoch=g["completion_epoch"], chunk_size=d.chunk_size)
            rpt = simulate(sched, t, d, SimOptions(switch_mode=mode))
            out[f"{name}/{vname}"] = {
                "case": name, "switch_mode": mode, "events": evs,
                "violations": [[v.kind, v.location, v.epoch] for v in rpt.violations],
                "completion_epoch": rpt.completion_epoch, "transfer_time": rpt.transfer_time,
                "per_entry": [[s, c, dst, k] for (s, c, dst), k in rpt.per_entry_completion.items()],
                "completion_epochs": [[dst, k] for dst, k in rpt.completion_epochs.items()],
            }
            print(name, vname, len(rpt.violations), rpt.completion_epoch, flush=True)
    with open(os.path.join(HERE, "sim_golden.json"), "w") as f:
        json.dump(out, f, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
