"""B200-native TE-CCL LP engine (arXiv 2305.13479 hot path).

Python entry points mirror the reference package `collsched` for the LP
path: topology + demand + epoch config in, device-built LP, GPU PDLP solve,
per-epoch flow schedule and finish time out. Heavy lifting lives in
libteccl_b200.so (csrc/), called through a plain C ABI (include/teccl_b200.h).
"""

from .checker import CheckReport, check_lp_schedule
from .demand import Demand, generate_demand, merge_demands
from .epochs import EpochConfig, compute_delta, epoch_duration
from .errors import (CollschedError, ConservationError, HorizonInfeasibleError,
                     ScheduleError, SolverBackendError, SolverTimeoutError, ValidationError)
from .lp import DeviceLP, LpPlan, ModelOptions, build_lp_model, lp_completion_epoch, make_plan
from .schedule import Schedule, ScheduleEvent, lp_rates_to_schedule
from .solver import Solution, SolverOptions, min_feasible_horizon, solve
from .topology import Edge, Topology, validate_topology
from .workflow import SynthesisResult, synthesize

__all__ = [
    "CheckReport", "check_lp_schedule", "Demand", "generate_demand", "merge_demands",
    "EpochConfig", "compute_delta", "epoch_duration", "CollschedError", "ConservationError",
    "HorizonInfeasibleError", "ScheduleError", "SolverBackendError", "SolverTimeoutError",
    "ValidationError", "DeviceLP", "LpPlan", "ModelOptions", "build_lp_model",
    "lp_completion_epoch", "make_plan", "Solution", "SolverOptions", "min_feasible_horizon",
    "solve", "Edge", "Topology", "validate_topology", "Schedule", "ScheduleEvent",
    "lp_rates_to_schedule", "SynthesisResult", "synthesize",
]
