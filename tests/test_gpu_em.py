"""Epoch-major matrix-free operator of row-partitioned LPs (te_gen.cuh EmOp):
every block's A.x / A^T.y, bounds and costs against the block's stored
CSR/CSC (built by the reference-faithful generators, themselves pinned to the
reference's golden fixtures), bit for bit; block solves with the operator."""

import ctypes as C

import numpy as np
import pytest

from paper_2305_13479_b200 import (EpochConfig, ModelOptions, SolverOptions, epoch_duration,
                                   generate_demand, make_plan)
from paper_2305_13479_b200 import _native as nat
from paper_2305_13479_b200.dist import build_partition
from paper_2305_13479_b200.errors import SolverBackendError
from paper_2305_13479_b200.solver import pdlp_options
from tests.golden.cases import CASES, build

pytestmark = pytest.mark.gpu


def _plan(name, phase1=False):
    from dataclasses import replace
    t, d, tau, K, blim = build(name)
    plan = make_plan(t, d, EpochConfig(tau, K, "fastest", 1, d.chunk_size),
                     ModelOptions(buffer_limit=blim))
    return replace(plan, phase1=True, _desc=None) if phase1 else plan


def _check_block(part, rng):
    i = part.info
    for transpose in (False, True):
        nin = (i["win_r1"] - i["win_r0"]) if transpose else (i["win_c1"] - i["win_c0"])
        v = rng.integers(-1000, 1000, nin).astype(np.float64)
        b = part.apply(v, transpose=transpose, matrix_free=0)
        a = part.apply(v, transpose=transpose, matrix_free=1)
        for k in a:
            assert np.array_equal(a[k], b[k]), (part.world, part.rank, transpose, k)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("phase1", [False, True])
def test_em_operator_equals_stored_blocks(name, phase1):
    plan = _plan(name, phase1)
    rng = np.random.default_rng(11)
    for world in (1, 2, 3):
        for rank in range(world):
            try:
                part = build_partition(plan, world, rank)
            except SolverBackendError as exc:  # horizon too short to split this many ways
                assert "too thin" in str(exc)
                continue
            _check_block(part, rng)
            part.close()


def test_em_operator_multichassis_blocks():
    # NDv2 4-chassis AllGather: init rows on rank 0, last rows / final buffers
    # on the last rank, halo windows in between
    from paper_2305_13479_b200.topology import ndv2
    t = ndv2(4)
    d = generate_demand("allgather", t, 1, 25000)
    plan = make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), 60, "fastest", 1, 25000))
    rng = np.random.default_rng(3)
    for world in (1, 4):
        for rank in range(world):
            part = build_partition(plan, world, rank)
            _check_block(part, rng)
            part.close()


def _solve_block(part, mf, eps=1e-8, max_iters=5_000_000):
    o = pdlp_options(SolverOptions(eps_rel=eps, max_iters=max_iters, pdlp={"matrix_free": mf}))
    n = part.info["own_c1"] - part.info["own_c0"]
    m = part.info["own_r1"] - part.info["own_r0"]
    x, y = np.empty(n), np.empty(m)
    res = nat.PdlpResult()
    nat.check(part.ctx.lib.teccl_pdlp_solve(part.ctx.handle, part.handle, C.byref(o),
                                            nat.ptr(x, C.c_double), nat.ptr(y, C.c_double),
                                            C.byref(res)))
    return res, x


def test_em_block_solve_matches_stored():
    # one block holding the whole LP (world 1): the matrix-free solve agrees
    # with the stored-matrix solve of the same epoch-major LP
    from paper_2305_13479_b200.topology import ndv2
    t = ndv2(2)
    d = generate_demand("allgather", t, 2, 25000)
    plan = make_plan(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), 530, "fastest", 1, 25000))
    part = build_partition(plan, 1, 0)
    r0, _ = _solve_block(part, 0)
    r1, x1 = _solve_block(part, 2)
    assert r0.status == r1.status == 0
    assert -r1.primal_obj == pytest.approx(-r0.primal_obj, rel=1e-6)
    assert part.step_bench(3, {"matrix_free": 2})["matrix_free"] == 2
    part.close()
