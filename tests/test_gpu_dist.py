"""Row-partitioned solve on 2 GPUs (one process per GPU, CUDA-IPC peer
exchange), compared with the single-GPU solve of the same LP. Skipped unless
two GPUs are visible -- two ranks must never share one GPU (their kernels
wait on each other)."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, mf):
    import torch.distributed as dist
    from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand
    from paper_2305_13479_b200.dist import solve_partitioned
    from paper_2305_13479_b200.topology import dgx1
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = dgx1()
        d = generate_demand("allgather", t, 1, 25000)
        cfg = EpochConfig(epoch_duration(t, 25000, "fastest", 1), 12, "fastest", 1, 25000)
        res = solve_partitioned(t, d, cfg, eps_rel=1e-8, device=rank, gather=True,
                                pdlp={"matrix_free": mf})
        out[rank] = (res["status"], res["objective"], res["iters"],
                     res["x"] if rank == 0 else None)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mf", [0, 2])  # stored SELL blocks, epoch-major matrix-free blocks
def test_two_gpu_partition_matches_one_gpu(mf):
    import torch.multiprocessing as mp
    from paper_2305_13479_b200 import (EpochConfig, SolverOptions, build_lp_model,
                                       check_lp_schedule, epoch_duration, generate_demand,
                                       lp_completion_epoch, solve)
    from paper_2305_13479_b200.topology import dgx1
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out, mf), nprocs=2, join=True)
    st0, obj0, it0, x = out[0]
    st1, obj1, it1, _ = out[1]
    assert st0 == st1 == "optimal" and obj0 == obj1 and it0 == it1
    t = dgx1()
    d = generate_demand("allgather", t, 1, 25000)
    cfg = EpochConfig(epoch_duration(t, 25000, "fastest", 1), 12, "fastest", 1, 25000)
    lp = build_lp_model(t, d, cfg)
    single = solve(lp, SolverOptions(eps_rel=1e-8))
    assert obj0 == pytest.approx(single.objective, rel=1e-6)
    rep = check_lp_schedule(lp.plan, x, tol=1e-5)
    assert rep.ok and rep.completion_epoch == lp_completion_epoch(single, tol=1e-5)


def _src_worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2305_13479_b200 import EpochConfig, epoch_duration, generate_demand
    from paper_2305_13479_b200.dist import solve_source_partitioned
    from paper_2305_13479_b200.topology import ndv2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = ndv2(2)
        d = generate_demand("allgather", t, 1, 25000)
        cfg = EpochConfig(epoch_duration(t, 25000, "fastest", 1), 270, "fastest", 1, 25000)
        res = solve_source_partitioned(t, d, cfg, eps_rel=1e-8, device=rank, gather=True)
        out[rank] = (res["status"], res["objective"], res["iters"], res["x"] if rank == 0 else None)
    finally:
        dist.destroy_process_group()


def _check_src(world):
    import torch.multiprocessing as mp
    from paper_2305_13479_b200 import (EpochConfig, SolverOptions, build_lp_model, check_lp_schedule,
                                       epoch_duration, generate_demand, lp_completion_epoch, solve)
    from paper_2305_13479_b200.topology import ndv2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_src_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    st = {out[r][0] for r in range(world)}
    objs = {out[r][1] for r in range(world)}
    its = {out[r][2] for r in range(world)}
    assert st == {"optimal"} and len(objs) == 1 and len(its) == 1  # identical decisions on every rank
    t = ndv2(2)
    d = generate_demand("allgather", t, 1, 25000)
    lp = build_lp_model(t, d, EpochConfig(epoch_duration(t, 25000, "fastest", 1), 270, "fastest", 1, 25000))
    single = solve(lp, SolverOptions(eps_rel=1e-8))
    assert out[0][1] == pytest.approx(single.objective, rel=1e-7)
    rep = check_lp_schedule(lp.plan, out[0][3], tol=1e-5)
    assert rep.ok and rep.completion_epoch == lp_completion_epoch(single, tol=1e-5)


def test_source_partition_one_rank():
    # world 1: the partitioned iteration (own-source kernels, capacity partials
    # through the exchange buffers) on one GPU
    _check_src(1)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_source_partition_two_gpus():
    _check_src(2)
