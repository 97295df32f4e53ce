# Per-iteration time of the configs[4] LP (32-chassis NDv2 AllGather,
# slowest-link epochs, K=2024) on N GPUs: two fixed-iteration runs (640 and
# 1920 iterations, never converging), device time difference / 1280.
#   bash tools/c4_periter.sh N
N=${1:-1}
export PDLP_OPTS='{"step_safety": 0.9, "eps_infeas": 0.0}'
for it in 640 1920; do
  if [ "$N" = 1 ]; then
    python - $it <<PY
import json, sys, os
sys.path.insert(0, os.getcwd())
from paper_2305_13479_b200 import EpochConfig, SolverOptions, epoch_duration, generate_demand, make_plan, solve
from paper_2305_13479_b200.lp import build_from_plan
from paper_2305_13479_b200.topology import ndv2
t = ndv2(32); d = generate_demand("allgather", t, 1, 25000)
lp = build_from_plan(make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "slowest", 1), 2024, "slowest", 1, 25000)))
o = json.loads(os.environ["PDLP_OPTS"])
sol = solve(lp, SolverOptions(eps_rel=1e-12, eps_res=0.0, max_iters=int(sys.argv[1]), time_limit=3000, pdlp=o))
print(json.dumps({"n_gpus": 1, "iters": sol.meta["iters"], "device_seconds_max": sol.meta["device_seconds"],
                  "cols": lp.num_vars}))
PY
  else
    torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + it % 97)) \
      tools/c4_solve.py 32 2024 slowest 1e-12 $it 0 2>/dev/null | grep '^{'
  fi
done
