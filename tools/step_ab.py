"""Per-launch time of the two half-step kernels (teccl_pdlp_step_bench) on
configs[1] and on the 16-chassis LP, for A/B of library variants
(TECCL_B200_LIB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload  # noqa: E402
from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand, make_plan  # noqa: E402
from paper_2305_13479_b200.lp import build_from_plan  # noqa: E402
from paper_2305_13479_b200.topology import ndv2  # noqa: E402

tag = os.path.basename(os.environ.get("TECCL_B200_LIB", "default"))
t, d, cfg = workload()
lps = {"c1": build_from_plan(make_plan(t, d, cfg))}
if os.environ.get("BIG", "1") == "1":
    t16 = ndv2(16)
    d16 = generate_demand("allgather", t16, 1, 25000)
    c16 = EpochConfig(epoch_duration(t16, 25000, "fastest", 1), 3860, "fastest", 1, 25000)
    lps["16ch"] = build_from_plan(make_plan(t16, d16, c16))
for name, lp in lps.items():
    reps = 200 if name == "c1" else 20
    sb = lp.step_bench(reps)
    sb2 = lp.step_bench(reps)
    print(tag, name, "col %.4f ms  row %.4f ms" % (min(sb["ms_col"], sb2["ms_col"]), min(sb["ms_row"], sb2["ms_row"])),
          flush=True)
    lp.close()
