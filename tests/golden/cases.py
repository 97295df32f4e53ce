"""Parity instances shared by the golden generator and the tests.

Each case is (topology, demand, tau, K, buffer_limit), built with this
package's generators; make_golden.py rebuilds the same instance with the
reference's own generators and asserts the two describe the same graph.
"""

from paper_2305_13479_b200.demand import Demand, generate_demand
from paper_2305_13479_b200.epochs import epoch_duration
from paper_2305_13479_b200.topology import (Edge, Topology, dgx1, dgx2, funnel, line, ndv2,
                                            relay_chain, ring, star)


def _fast_tau(t, d):
    return epoch_duration(t, d.chunk_size, "fastest", 1)


def build(name, mod=None):
    """Instance `name`; `mod` is a module namespace providing the same
    generator/type names (this package by default, the reference for goldens)."""
    if mod is None:
        import paper_2305_13479_b200.topology as topo
        import paper_2305_13479_b200.demand as dem
        import paper_2305_13479_b200.epochs as ep
        mod = {"topo": topo, "dem": dem, "ep": ep}
    topo, dem, ep = mod["topo"], mod["dem"], mod["ep"]
    fast = lambda t, d: ep.epoch_duration(t, d.chunk_size, "fastest", 1)
    if name == "ring2_a2a_K1":
        t = topo.ring(2); d = dem.generate_demand("alltoall", t, 1, 1); return t, d, 1.0, 1, None
    if name == "chain_K8":
        t = topo.relay_chain(1.0, 5.0)
        d = dem.Demand(frozenset({("s1", 0, "d"), ("s2", 1, "d")}), 2, 1); return t, d, 1.0, 8, None
    if name == "single_edge_K2":
        t = topo.Topology((0, 1), frozenset(), (topo.Edge(0, 1, 1.0),))
        d = dem.Demand(frozenset({(0, 0, 1)}), 1, 1); return t, d, 1.0, 2, None
    if name == "parallel_K2":
        t = topo.Topology(("s", "a", "b", "d"), frozenset(), (
            topo.Edge("s", "a", 0.5), topo.Edge("s", "b", 0.5),
            topo.Edge("a", "d", 0.5), topo.Edge("b", "d", 0.5)))
        d = dem.Demand(frozenset({("s", 0, "d")}), 1, 1); return t, d, 1.0, 2, None
    if name == "ring4_a2a2_K4":
        t = topo.ring(4); d = dem.generate_demand("alltoall", t, 2, 1); return t, d, 1.0, 4, None
    if name in ("dgx1_ag1_K8", "dgx1_ag1_K10", "dgx1_ag1_K6"):
        t = topo.dgx1(); d = dem.generate_demand("allgather", t, 1, 25000)
        return t, d, fast(t, d), int(name.split("K")[-1]), None
    if name == "dgx1_a2a1_K8":
        t = topo.dgx1(); d = dem.generate_demand("alltoall", t, 1, 25000); return t, d, fast(t, d), 8, None
    if name == "ndv2x2_ag1_K24":
        t = topo.ndv2(2); d = dem.generate_demand("allgather", t, 1, 25000); return t, d, fast(t, d), 24, None
    if name == "star3_K5":
        t = topo.star(3)
        d = dem.Demand(frozenset({("s", 0, "d1"), ("s", 0, "d2"), ("s", 0, "d3")}), 1, 1)
        return t, d, 1.0, 5, None
    if name == "funnel_blimit_K4":
        t = topo.funnel()
        d = dem.Demand(frozenset({("s1", 0, "d"), ("s2", 1, "d"), ("s3", 2, "d")}), 3, 1)
        return t, d, 1.0, 4, 3.0
    if name == "override_K3":
        base = topo.line(3)
        t = topo.Topology(base.nodes, base.switches, base.edges, {(0, 1, 1): 0.5})
        d = dem.generate_demand("allgather", t, 1, 1); return t, d, 1.0, 3, None
    if name == "dgx2x1_a2a_K20":
        t = topo.dgx2(1); d = dem.generate_demand("alltoall", t, 1, 25000); return t, d, fast(t, d), 20, None
    raise KeyError(name)


CASES = ["ring2_a2a_K1", "chain_K8", "single_edge_K2", "parallel_K2", "ring4_a2a2_K4",
         "dgx1_ag1_K6", "dgx1_ag1_K8", "dgx1_ag1_K10", "dgx1_a2a1_K8", "ndv2x2_ag1_K24",
         "star3_K5", "funnel_blimit_K4", "override_K3", "dgx2x1_a2a_K20"]
