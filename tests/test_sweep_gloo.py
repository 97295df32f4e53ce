"""Multi-process sweep plumbing on CPU: world_size 2 over gloo (no GPU).
The solver is replaced by a pure function so only sharding/gathering runs."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_13479_b200.sweep import Instance, default_sweep, run_sweep, shard


def _fake_solver(inst, device, slot=0):
    return {"instance": inst.chunk_size * 10 + inst.em, "device": device, "slot": slot}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        recs = run_sweep(default_sweep(), rank, world, device=rank, solver=_fake_solver, streams=3)
        out[rank] = recs
    finally:
        dist.destroy_process_group()


def test_default_sweep_shape():
    s = default_sweep()
    assert len(s) == 64 and len(set(s)) == 64
    assert sorted(shard(list(range(10)), 1, 4)) == [1, 5, 9]
    assert sum(len(shard(s, r, 8)) for r in range(8)) == 64


def test_gloo_two_ranks_gather_in_order():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    expect = [_fake_solver(inst, 0)["instance"] for inst in default_sweep()]
    for rank in range(world):
        recs = out[rank]
        assert [r["instance"] for r in recs] == expect
        # every instance solved exactly once, on the rank that owns it
        assert [r["device"] for r in recs] == [i % world for i in range(64)]


def test_concurrent_streams_keep_order_and_use_every_slot():
    import time
    from paper_2305_13479_b200.sweep import solve_shard

    def slow(inst, device, slot=0):
        time.sleep(0.01)
        return _fake_solver(inst, device, slot)

    items = list(enumerate(default_sweep()[:24]))
    recs = solve_shard(items, 0, slow, streams=4)
    assert [i for i, _ in recs] == list(range(24))
    assert [r["instance"] for _, r in recs] == [_fake_solver(x, 0)["instance"] for _, x in items]
    assert {r["slot"] for _, r in recs} == {0, 1, 2, 3}
