"""ctypes binding of libteccl_b200.so (declared in include/teccl_b200.h).

The product path has no CPU fallback: if the library is missing or no sm_100
device is present, every entry point raises SolverBackendError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import SolverBackendError

LIB_NAME = "libteccl_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# Every symbol include/teccl_b200.h declares (tests check the export table).
EXPORTED = (
    "teccl_last_error", "teccl_version", "teccl_ctx_create", "teccl_ctx_destroy",
    "teccl_ctx_sync", "teccl_lp_build_te", "teccl_lp_build_te_part", "teccl_dist_export",
    "teccl_dist_connect", "teccl_src_setup", "teccl_src_export", "teccl_src_connect", "teccl_lp_from_csr", "teccl_lp_dims",
    "teccl_lp_export", "teccl_lp_export_csc", "teccl_lp_destroy",
    "teccl_pdlp_default_opts", "teccl_pdlp_solve", "teccl_pdlp_solve_dev",
    "teccl_spmv_bench", "teccl_pdlp_step_bench", "teccl_pdlp_step_bench_opts", "teccl_lp_apply", "teccl_check_te", "teccl_check_te_dev",
    "teccl_schedule_te", "teccl_schedule_fetch", "teccl_simulate", "teccl_simulate_fetch",
)

STATUS = {0: "optimal", 1: "iteration-limit", 2: "time-limit", 3: "primal-infeasible",
          4: "numerical", 5: "peer-timeout"}

_p = C.POINTER


class TeDesc(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32), ("num_edges", C.c_int32), ("num_sources", C.c_int32),
        ("num_pairs", C.c_int32), ("K", C.c_int32),
        ("node_is_switch", _p(C.c_uint8)), ("edge_src", _p(C.c_int32)),
        ("edge_dst", _p(C.c_int32)), ("edge_delta", _p(C.c_int32)),
        ("edge_cap", _p(C.c_double)), ("source_node", _p(C.c_int32)),
        ("pair_source", _p(C.c_int32)), ("pair_dst", _p(C.c_int32)),
        ("pair_units", _p(C.c_double)), ("buffer_limit", C.c_double),
        ("phase1", C.c_int32),
    ]


class PdlpOpts(C.Structure):
    _fields_ = [
        ("eps_rel", C.c_double), ("max_iters", C.c_int64), ("time_limit", C.c_double),
        ("check_every", C.c_int32), ("ruiz_iters", C.c_int32), ("lookahead", C.c_int32),
        ("verbose", C.c_int32), ("reflection", C.c_double), ("use_graphs", C.c_int32),
        ("warm_start", C.c_int32), ("restart_sufficient", C.c_double),
        ("restart_necessary", C.c_double), ("restart_artificial", C.c_double),
        ("omega_theta", C.c_double), ("omega_scale", C.c_double),
        ("omega_ki", C.c_double), ("omega_kd", C.c_double), ("col_pipeline", C.c_int32),
        ("matrix_free", C.c_int32), ("pdl", C.c_int32),
        ("fused_halo", C.c_int32), ("eps_res", C.c_double), ("eps_infeas", C.c_double),
        ("infeas_every", C.c_int32), ("persist", C.c_int32),
        ("omega_bias", C.c_double), ("step_safety", C.c_double),
    ]


class PdlpResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("restarts", C.c_int32), ("iters", C.c_int64),
        ("primal_obj", C.c_double), ("dual_obj", C.c_double), ("rel_gap", C.c_double),
        ("rel_primal_res", C.c_double), ("rel_dual_res", C.c_double),
        ("solve_seconds", C.c_double), ("omega", C.c_double), ("step", C.c_double),
        ("spmv_launches", C.c_int64), ("infeas_cert", C.c_double),
    ]


class SimDesc(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32), ("node_is_switch", _p(C.c_uint8)), ("num_edges", C.c_int32),
        ("edge_delta", _p(C.c_int32)), ("edge_window", _p(C.c_int32)),
        ("edge_budget", _p(C.c_double)), ("num_entries", C.c_int64),
        ("entry_source", _p(C.c_int32)), ("entry_chunk", _p(C.c_int32)),
        ("entry_dst", _p(C.c_int32)), ("switch_mode", C.c_int32), ("tolerance", C.c_double),
    ]


class CheckReport(C.Structure):
    _fields_ = [
        ("capacity_violations", C.c_int64), ("causality_violations", C.c_int64),
        ("switch_violations", C.c_int64), ("unmet_pairs", C.c_int64),
        ("completion_epoch", C.c_int32), ("max_capacity_excess", C.c_int64),
        ("max_buffer_deficit", C.c_int64),
    ]


_lib = None
_lock = threading.Lock()
_ctx_lock = threading.Lock()


def load(path: str | None = None):
    """Load the shared library and declare signatures; raises if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or os.environ.get("TECCL_B200_LIB", LIB_PATH)
        if not os.path.exists(p):
            raise SolverBackendError(
                f"{LIB_NAME} not built at {p}; run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = C.CDLL(p)
        except OSError as exc:
            raise SolverBackendError(f"cannot load {p}: {exc}") from exc
        vp = C.c_void_p
        sig = {
            "teccl_last_error": (C.c_char_p, []),
            "teccl_version": (C.c_char_p, []),
            "teccl_ctx_create": (C.c_int, [C.c_int, _p(vp)]),
            "teccl_ctx_destroy": (C.c_int, [vp]),
            "teccl_ctx_sync": (C.c_int, [vp]),
            "teccl_lp_build_te": (C.c_int, [vp, _p(TeDesc), _p(vp)]),
            "teccl_lp_build_te_part": (C.c_int, [vp, _p(TeDesc), C.c_int32, C.c_int32, _p(vp),
                                                 _p(C.c_int64)]),
            "teccl_dist_export": (C.c_int, [vp, vp, _p(C.c_uint8), _p(C.c_int64)]),
            "teccl_dist_connect": (C.c_int, [vp, vp, _p(C.c_uint8), C.c_int64]),
            "teccl_src_setup": (C.c_int, [vp, vp, C.c_int32, C.c_int32, _p(C.c_int64)]),
            "teccl_src_export": (C.c_int, [vp, vp, _p(C.c_uint8), _p(C.c_int64)]),
            "teccl_src_connect": (C.c_int, [vp, vp, _p(C.c_uint8), C.c_int64]),
            "teccl_lp_from_csr": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int64, _p(C.c_int64),
                                            _p(C.c_int32), _p(C.c_double), _p(C.c_double),
                                            _p(C.c_double), _p(C.c_double), _p(C.c_double),
                                            _p(C.c_double), _p(vp)]),
            "teccl_lp_dims": (C.c_int, [vp, _p(C.c_int32), _p(C.c_int32), _p(C.c_int64)]),
            "teccl_lp_export": (C.c_int, [vp, _p(C.c_int64), _p(C.c_int32), _p(C.c_double),
                                          _p(C.c_double), _p(C.c_double), _p(C.c_double),
                                          _p(C.c_double), _p(C.c_double)]),
            "teccl_lp_export_csc": (C.c_int, [vp, _p(C.c_int64), _p(C.c_int32), _p(C.c_double)]),
            "teccl_lp_destroy": (C.c_int, [vp]),
            "teccl_pdlp_default_opts": (None, [_p(PdlpOpts)]),
            "teccl_pdlp_solve": (C.c_int, [vp, vp, _p(PdlpOpts), _p(C.c_double), _p(C.c_double),
                                           _p(PdlpResult)]),
            "teccl_pdlp_solve_dev": (C.c_int, [vp, vp, _p(PdlpOpts), vp, vp, _p(PdlpResult)]),
            "teccl_spmv_bench": (C.c_int, [vp, vp, C.c_int32, _p(C.c_double), _p(C.c_double)]),
            "teccl_pdlp_step_bench": (C.c_int, [vp, vp, C.c_int32, _p(C.c_double)]),
            "teccl_pdlp_step_bench_opts": (C.c_int, [vp, vp, vp, C.c_int32, _p(C.c_double)]),
            "teccl_lp_apply": (C.c_int, [vp, vp, C.c_int32, C.c_int32, _p(C.c_double), _p(C.c_double),
                                         _p(C.c_double), _p(C.c_double), _p(C.c_double)]),
            "teccl_check_te": (C.c_int, [vp, _p(TeDesc), _p(C.c_double), C.c_int64, C.c_int64,
                                         _p(CheckReport)]),
            "teccl_check_te_dev": (C.c_int, [vp, _p(TeDesc), vp, C.c_int64, C.c_int64,
                                             _p(CheckReport)]),
            "teccl_schedule_te": (C.c_int, [_p(TeDesc), _p(C.c_double), C.c_double, C.c_double,
                                            _p(C.c_int32), _p(C.c_int32), _p(C.c_int32),
                                            _p(C.c_int32), _p(C.c_int32), _p(C.c_int32),
                                            _p(C.c_int32), C.c_int32, _p(vp), _p(C.c_int64)]),
            "teccl_schedule_fetch": (C.c_int, [vp, _p(C.c_int32), _p(C.c_int32), _p(C.c_int32),
                                               _p(C.c_int32), _p(C.c_double)]),
            "teccl_simulate": (C.c_int, [_p(SimDesc), C.c_int64, _p(C.c_int32), _p(C.c_int32),
                                         _p(C.c_int32), _p(C.c_int32), _p(C.c_int32), _p(C.c_int32),
                                         _p(C.c_double), _p(C.c_int32), _p(C.c_int32), C.c_int32,
                                         _p(vp), _p(C.c_int64)]),
            "teccl_simulate_fetch": (C.c_int, [vp, _p(C.c_int64), _p(C.c_int64), _p(C.c_int64),
                                               _p(C.c_int32)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.teccl_last_error().decode() if _lib is not None else "?"
        raise SolverBackendError(f"teccl_b200 error {rc}: {msg}")


def ptr(arr, ctype):
    """Pointer into a contiguous numpy array (caller keeps `arr` alive)."""
    return arr.ctypes.data_as(C.POINTER(ctype))


class Context:
    """One device + one stream. Created lazily per device and reused."""

    _cache: dict = {}

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.teccl_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: int = 0, slot: int = 0) -> "Context":
        """Context `slot` of `device` (slot > 0: extra streams for concurrent
        independent solves on one GPU)."""
        with _ctx_lock:
            ctx = cls._cache.get((device, slot))
            if ctx is None:
                ctx = cls._cache[(device, slot)] = Context(device)
        return ctx

    def sync(self) -> None:
        check(self.lib.teccl_ctx_sync(self.handle))
