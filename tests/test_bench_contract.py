"""bench.py's contract pieces that need no GPU: both arms print the same
`config` object, and the workloads are the LPs DESIGN.md quotes (configs[1]
and the configs[4] flagship)."""

import bench
from paper_2305_13479_b200 import make_plan


def test_both_arms_share_the_config_object():
    t, d, cfg = bench.workload()
    c = bench.bench_config(cfg)
    assert c == bench.bench_config(cfg)  # built by one function for both arms
    assert c["K"] == 530 and c["eps_rel"] == 1e-4 and c["eps_res"] == 1e-6
    assert set(c) == {"workload", "K", "eps_rel", "eps_res", "criterion", "l2"}


def test_headline_lp_shape():
    t, d, cfg = bench.workload()
    p = make_plan(t, d, cfg)
    assert (p.num_vars, p.num_rows) == (966_976, 307_656)


def test_flagship_lp_shape(monkeypatch):
    monkeypatch.delenv("BENCH_FLAGSHIP_CHASSIS", raising=False)
    t, d, cfg = bench.flagship_workload()
    p = make_plan(t, d, cfg)
    assert cfg.K == 2024 and cfg.duration_mode == "slowest"
    assert (p.num_vars, p.num_rows) == (960_704_512, 267_557_376)
    assert len(t.gpus) == 256
