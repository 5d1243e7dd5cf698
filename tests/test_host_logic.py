"""CPU: host-side logic of the drop-in that runs before any device call —
placement validation with the reference's exact ValidationError texts
(flow_graph.cpp:52-61), the cluster model (cluster.cpp:62-100), cluster
validation (cluster.cpp:237-300), and the hybrid library's linkage (the
reference planner resolving build_flow_graph / max_flow to this repo)."""

import ctypes
import json
import os
import subprocess

import pytest

import paper_2406_01566_b200 as h
from paper_2406_01566_b200.clusters import chain_cluster, het42, make_link, make_node
from _support import HYB_SO, Oracle


def C(d):
    return h.Cluster.from_json(json.dumps(d))


def test_invalid_placements_raise_reference_messages_before_any_device_call():
    c = C(chain_cluster(2, 2, 1000.0))
    with pytest.raises(h.ValidationError, match=r"^placement references unknown node 'zz'$"):
        h.build_flow_graph(c, {"zz": (0, 2)}, False)
    with pytest.raises(h.ValidationError, match=r"^placement for 'n0' outside \[0, 4\)$"):
        h.max_flow_value(c, {"n0": (0, 5)})
    with pytest.raises(h.ValidationError, match=r"^placement for 'n0' exceeds its VRAM layer capacity$"):
        h.plan_for_placement(c, {"n0": (0, 3)})
    # first failing node in id order decides (the reference iterates a std::map)
    with pytest.raises(h.ValidationError, match="'n0'"):
        h.max_flow_value(c, {"n1": (0, 9), "n0": (-1, 1)})


def test_cluster_model_matches_the_oracle():
    d = het42()
    c = C(d)
    o = Oracle(d)
    assert [c.max_layers(i) for i in c.node_ids] == o.kmax()
    # compute_edge_capacity validates j before touching the device (cluster.cpp:70-73)
    with pytest.raises(h.ValidationError, match="outside profile range: j=0"):
        c.compute_edge_capacity("a100-0", 0)
    with pytest.raises(h.ValidationError, match="outside profile range: j=12"):
        c.compute_edge_capacity("a100-0", 12)


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d["links"].append(dict(d["links"][0])), "duplicate link"),
    (lambda d: d["nodes"].append(dict(d["nodes"][0])), "duplicate node id"),
    (lambda d: d["nodes"][0].update(kv_reserve=1.0), "kv_reserve must be in"),
    (lambda d: d["links"].append(make_link("n0", "ghost", 1e9)), "is not a declared node"),
    (lambda d: d["links"].append(make_link("n1", "n1", 1e9)), "self-link"),
    (lambda d: d["model"].update(num_layers=99, param_gb=99.0), "insufficient VRAM"),
    (lambda d: d["nodes"][0].update(throughput_table={"1": 5.0}), "exactly one of"),
])
def test_validate_cluster_errors(mutate, msg):
    d = chain_cluster(2, 2, 1000.0)
    mutate(d)
    with pytest.raises(h.ValidationError, match=msg):
        C(d)


def test_parse_errors():
    d = chain_cluster(2, 2, 1000.0)
    d["model"]["num_layers"] = "four"
    with pytest.raises(h.ParseError, match="must be a number"):
        C(d)
    with pytest.raises(h.ParseError, match="invalid JSON"):
        h.Cluster.from_json("{nope")


def test_plan_json_round_trip_on_host():
    plan = h.Plan.from_json(json.dumps({
        "method": "custom", "status": "feasible", "objective": 450.0, "allow_partial": True,
        "nodes": [{"id": "n0", "start": 0, "end": 2}],
        "edges": [{"src": "coord", "dst": "n0", "flow": 450.0, "exec_start": 0, "exec_end": 2}]}))
    again = h.Plan.from_json(plan.to_json())
    assert again.to_json() == plan.to_json()
    assert again.edges == [("coord", "n0", 450.0, 0, 2)] and again.placement == {"n0": (0, 2)}


@pytest.mark.skipif(not os.path.exists(HYB_SO), reason="hybrid library not built")
def test_hybrid_library_links_the_reference_planner_to_this_flow_graph():
    lib = ctypes.CDLL(HYB_SO)
    assert hasattr(lib, "hyb_plan_milp")
    syms = subprocess.run(["nm", "-D", "--defined-only", HYB_SO], capture_output=True, text=True).stdout
    # build_flow_graph / max_flow are defined by shim_flow.o (not the reference's
    # flow_graph.o), and the engine they call is this repo's libhelio_gpu.so
    assert "_ZN5helio8max_flowERNS_9FlowGraphE" in syms
    assert "helio_gpu_set_cluster" not in syms  # resolved from libhelio_gpu.so
    needed = subprocess.run(["readelf", "-d", HYB_SO], capture_output=True, text=True).stdout
    assert "libhelio_gpu.so" in needed
