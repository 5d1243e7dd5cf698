"""GPU: the reference's own hot-path test cases, re-expressed against the
drop-in (proj/tests/test_flow.cpp, test_scheduler.cpp, test_placement.cpp:65-84,
tests/python/test_smoke.py:76-81).  Same clusters (test_support.hpp), same
expectations."""

import json

import numpy as np
import pytest

import paper_2406_01566_b200 as h
from paper_2406_01566_b200.clusters import chain_cluster, make_link, make_node

pytestmark = pytest.mark.gpu


def C(d):
    return h.Cluster.from_json(json.dumps(d))


def toy(L, nodes, links):
    return {"model": {"name": "toy", "num_layers": L, "param_gb": float(L)},
            "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def test_two_stage_chain_bottlenecked_by_compute():  # test_flow.cpp:15-34
    c = C(chain_cluster(2, 2, 1000.0))
    g = h.build_flow_graph(c, {"n0": (0, 2), "n1": (2, 4)}, False)
    assert g.num_vertices == 6 and len(g.edges) == 5
    assert h.max_flow(g) == pytest.approx(500.0)
    net = np.zeros(g.num_vertices)
    for (u, v, cap, flow, kind, *_rest) in g.edges:
        net[u] -= flow
        net[v] += flow
    for x in range(g.num_vertices):
        if x not in (g.source, g.sink):
            assert abs(net[x]) <= 1e-12


def test_parallel_full_model_replicas_add():  # test_flow.cpp:36-48
    c = C(toy(2, [make_node("a", 2, 600.0), make_node("b", 2, 400.0)],
              [make_link("coord", "a", 10e9), make_link("coord", "b", 10e9),
               make_link("a", "coord", 10e9), make_link("b", "coord", 10e9)]))
    assert h.max_flow_value(c, {"a": (0, 2), "b": (0, 2)}, False) == pytest.approx(500.0)


def test_overlapping_stages_partial_only():  # test_flow.cpp:50-78
    c = C(toy(4, [make_node("a", 3, 900.0), make_node("b", 3, 600.0)],
              [make_link("coord", "a", 10e9), make_link("a", "b", 10e9), make_link("b", "coord", 10e9)]))
    p = {"a": (0, 3), "b": (1, 4)}
    assert h.max_flow_value(c, p, False) == pytest.approx(0.0)
    assert h.max_flow_value(c, p, True) == pytest.approx(200.0)
    g = h.build_flow_graph(c, p, True)
    inter = [e for e in g.edges if e[4] == 3]
    assert len(inter) == 1
    u, v, cap, flow, kind, src, dst, es, ee = inter[0]
    assert (src, dst, es, ee) == ("a", "b", 3, 4)


def test_exec_intervals_on_coordinator_edges():  # test_flow.cpp:80-93
    c = C(chain_cluster(2, 2, 1000.0))
    g = h.build_flow_graph(c, {"n0": (0, 2), "n1": (2, 4)}, False)
    for (u, v, cap, flow, kind, src, dst, es, ee) in g.edges:
        if kind == 1:
            assert (es, ee) == (0, 2)
        elif kind == 2:
            assert (es, ee) == (4, 4)


def test_slow_nic_clamps_compute_edge():  # test_flow.cpp:95-104
    d = chain_cluster(1, 2, 1000.0)
    d["nodes"][0]["nic_in_gbps"] = 0.001  # 1 Mbps
    c = C(d)
    assert c.compute_edge_capacity("n0", 2) == pytest.approx(1e6 / (8.0 * 16384.0))
    c2 = C(chain_cluster(1, 2, 1000.0))
    assert c2.compute_edge_capacity("n0", 2) == pytest.approx(500.0)


def test_no_span_and_empty_carry_no_flow():  # test_flow.cpp:106-115
    c = C(chain_cluster(2, 2, 1000.0))
    assert h.max_flow_value(c, {"n0": (0, 2)}, False) == 0.0
    assert h.max_flow_value(c, {}, False) == 0.0


def test_invalid_placements_rejected():  # test_flow.cpp:117-122
    c = C(chain_cluster(2, 2, 1000.0))
    with pytest.raises(h.ValidationError, match="unknown node 'zz'"):
        h.build_flow_graph(c, {"zz": (0, 2)}, False)
    with pytest.raises(h.ValidationError, match=r"outside \[0, 4\)"):
        h.build_flow_graph(c, {"n0": (0, 5)}, False)
    with pytest.raises(h.ValidationError, match="VRAM layer capacity"):
        h.build_flow_graph(c, {"n0": (0, 3)}, False)


def test_batched_status_codes():
    c = C(chain_cluster(2, 2, 1000.0))
    e = h.Engine(c)
    rows = np.array([[[0, 2], [2, 4]], [[0, 5], [2, 4]], [[0, 3], [2, 4]], [[-1, 2], [2, 4]],
                     [[3, 1], [2, 4]]], np.int16)
    v, s = e.score(rows, False)
    assert list(s) == [0, 2, 3, 2, 0]
    assert v[0] == 500.0 and v[4] == 0.0


def test_min_cut_isolates_bottleneck():  # test_flow.cpp:124-139
    d = chain_cluster(2, 2, 1000.0)
    d["nodes"][1]["peak_layer_tokens_per_s"] = 400.0
    c = C(d)
    g = h.build_flow_graph(c, {"n0": (0, 2), "n1": (2, 4)}, False)
    assert h.max_flow(g) == pytest.approx(200.0)
    side = set(g.min_cut_source_side())
    assert g.source in side and g.sink not in side
    cut = sum(cap for (u, v, cap, *_r) in g.edges if u in side and v not in side)
    assert cut == pytest.approx(200.0)


def test_smoke_max_flow_matches_manual_placement():  # test_smoke.py:76-81
    d = {"model": {"name": "tiny", "num_layers": 4, "param_gb": 4},
         "coordinator": {"id": "coord"},
         "nodes": [{"id": "a", "vram_gb": 9, "peak_layer_tokens_per_s": 1200},
                   {"id": "b", "vram_gb": 9, "peak_layer_tokens_per_s": 800}],
         "links": [{"src": "coord", "dst": "a", "bandwidth_mbps": 1000, "latency_ms": 1},
                   {"src": "coord", "dst": "b", "bandwidth_mbps": 1000, "latency_ms": 1},
                   {"src": "a", "dst": "coord", "bandwidth_mbps": 1000, "latency_ms": 1},
                   {"src": "b", "dst": "coord", "bandwidth_mbps": 1000, "latency_ms": 1},
                   {"src": "a", "dst": "b", "bandwidth_mbps": 1000, "latency_ms": 1}]}
    c = C(d)
    assert h.max_flow_value(c, {"a": (0, 4), "b": (0, 4)}) == pytest.approx(500.0, rel=1e-9)
    assert h.max_flow_value(c, {"a": (0, 2), "b": (2, 4)}) == pytest.approx(400.0, rel=1e-9)


def test_plan_edges_carry_objective_out_of_coordinator():  # test_placement.cpp:65-84
    c = C(chain_cluster(3, 2, 900.0))
    p = h.plan_for_placement(c, {"n0": (0, 2), "n1": (2, 4), "n2": (4, 6)})
    assert p.objective == pytest.approx(450.0)
    out = sum(f for (s, d, f, es, ee) in p.edges if s == "coord")
    assert out == pytest.approx(p.objective)


def test_iwrr_picker_interleaves_by_weight():  # test_scheduler.cpp:41-48
    p = h.IwrrPicker([3, 1, 2])
    assert p.next_all(12) == [0, 1, 2, 0, 2, 0, 0, 1, 2, 0, 2, 0]


def test_iwrr_picker_forfeits_masked_slots():  # test_scheduler.cpp:50-60
    p = h.IwrrPicker([3, 1, 2])
    seq = [p.next(lambda i: i != 0) for _ in range(6)]
    assert seq == [1, 2, 2, 1, 2, 2]
    assert p.next(lambda i: False) == -1
    assert p.next(lambda i: i != 0) != -1


def test_iwrr_weights_known_answers():  # test_scheduler.cpp:62-68
    assert h.iwrr_weights([2.0, 1.0]) == [32, 16]
    assert h.iwrr_weights([1000.0, 381.47]) == [32, 12]
    assert h.iwrr_weights([0.0001]) == [1]
    assert h.iwrr_weights([0.002, 0.001]) == [2, 1]
    assert h.iwrr_weights([5.0, 0.0001]) == [32, 1]


def y_plan(fa, fb):
    return h.Plan.from_json(json.dumps({
        "method": "milp", "status": "feasible", "objective": fa + fb, "allow_partial": True,
        "nodes": [{"id": "a", "start": 0, "end": 2}, {"id": "b", "start": 0, "end": 2}],
        "edges": [{"src": "coord", "dst": "a", "flow": fa, "exec_start": 0, "exec_end": 2},
                  {"src": "coord", "dst": "b", "flow": fb, "exec_start": 0, "exec_end": 2},
                  {"src": "a", "dst": "coord", "flow": fa, "exec_start": 2, "exec_end": 2},
                  {"src": "b", "dst": "coord", "flow": fb, "exec_start": 2, "exec_end": 2}]}))


def y_cluster():
    return C(toy(2, [make_node("a", 2, 600.0), make_node("b", 2, 400.0)],
                 [make_link("coord", "a", 10e9), make_link("coord", "b", 10e9),
                  make_link("a", "coord", 10e9), make_link("b", "coord", 10e9)]))


def test_admission_frequency_follows_plan_flows():  # test_scheduler.cpp:76-92
    c = y_cluster()
    routes = h.route_requests(c, y_plan(2.0, 1.0), [100] * 3000, [100] * 3000)
    assert all(r is not None and len(r) == 1 for r in routes)
    a = sum(1 for r in routes if r[0][0] == "a")
    assert abs(a / 3000 - 2.0 / 3.0) < 0.02


def test_multi_hop_routes_tile_the_layer_range():  # test_scheduler.cpp:128-161
    c = C(toy(6, [make_node("a", 3, 600.0), make_node("b", 3, 500.0)],
              [make_link("coord", "a", 10e9), make_link("a", "b", 10e9), make_link("b", "coord", 10e9)]))
    plan = h.Plan.from_json(json.dumps({
        "method": "milp", "status": "feasible", "objective": 1.5, "allow_partial": True,
        "nodes": [{"id": "a", "start": 0, "end": 3}, {"id": "b", "start": 3, "end": 6}],
        "edges": [{"src": "coord", "dst": "a", "flow": 1.5, "exec_start": 0, "exec_end": 3},
                  {"src": "a", "dst": "b", "flow": 1.5, "exec_start": 3, "exec_end": 6},
                  {"src": "b", "dst": "coord", "flow": 1.5, "exec_start": 6, "exec_end": 6}]}))
    (route,) = h.route_requests(c, plan, [50], [100])
    assert route == [("a", 0, 3), ("b", 3, 6)]


def test_scheduler_rejects_unusable_plans():  # test_scheduler.cpp:223-233
    c = y_cluster()
    empty = h.Plan.from_json(json.dumps({"method": "milp", "status": "feasible", "objective": 0,
                                         "allow_partial": True,
                                         "nodes": [{"id": "a", "start": 0, "end": 2}], "edges": []}))
    with pytest.raises(h.ValidationError):
        h.route_requests(c, empty, [1], [1])
    ghost = json.loads(y_plan(1.0, 1.0).to_json())
    ghost["edges"].append({"src": "coord", "dst": "zz", "flow": 1.0, "exec_start": 0, "exec_end": 2})
    with pytest.raises(h.ValidationError):
        h.route_requests(c, h.Plan.from_json(json.dumps(ghost)), [1], [1])
