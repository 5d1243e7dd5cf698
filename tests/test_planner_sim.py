"""The reference's host planner and simulator over this engine
(lib/libhelio_planner.so, include/helio_planner.h), the stateful Scheduler
drop-in (csrc/shim_sched.cpp), and the plan / report formats (SURVEY.md §8(b),
§8(f) ranks 2-4).

CPU tests: plan and cluster JSON are byte-identical to the reference's
serializers and cross-load both ways; prune_links; policy validation.
GPU tests (-m gpu): Scheduler admit/complete interleavings, simulate(), plan(c,
"milp"), plan edges and DOT reports, all against the pure reference
(oracle/_ref/libhelio_ref.so) on the same inputs."""

import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
from _support import RefCluster, bits, golden, golden_cluster, ref, ref_available, ref_trace

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
PLANNER = os.path.join(os.path.dirname(h.__file__), "lib", "libhelio_planner.so")
needs_planner = pytest.mark.skipif(not os.path.exists(PLANNER), reason="lib/libhelio_planner.so not built")

_i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

ROUTE_FIXTURES = {"route_geo24": "geo24_float", "route_fan3": "fan3", "route_kvmask": "kvmask"}


def _lib():
    lib = ref()
    if not getattr(lib, "_planner_sigs", False):
        lib.refh_plan_json.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_char_p, C.c_char_p, C.c_int]
        lib.refh_plan_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        lib.refh_to_dot.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_char_p, C.c_int, _i32p,
                                    C.POINTER(C.c_int)]
        lib.refh_sched_ops.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_uint64, C.c_int64, _i32p, _i64p, _i32p,
                                       C.c_int, _i32p, _i32p, _i32p, _i32p, C.c_char_p, _f64p, _f64p,
                                       C.c_char_p, C.c_int]
        lib.refh_simulate.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_int64, _f64p, _i32p, _i32p, C.c_int,
                                      C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_char_p, C.c_int]
        lib.refh_prune_json.argtypes = [C.c_void_p, C.c_double, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        lib._planner_sigs = True
    return lib


def _text(fn, *args, size=1 << 22):
    buf = C.create_string_buffer(size)
    n = fn(*args, buf, size)
    assert n >= 0, buf.value.decode()
    return buf.value.decode()


def _placement(d, row):
    return {d["nodes"][k]["id"]: (int(row[k, 0]), int(row[k, 1]))
            for k in range(len(d["nodes"])) if row[k, 1] > row[k, 0]}


def _cluster(d):
    return h.Cluster.from_json(json.dumps(d))


def ref_plan_json(d, row, method="custom", partial=True):
    rc = RefCluster(d)
    return _text(_lib().refh_plan_json, rc.h, np.ascontiguousarray(row, np.int16), int(partial), method.encode())


# --- formats (CPU) -------------------------------------------------------------

@needs_ref
@pytest.mark.parametrize("tag", sorted(ROUTE_FIXTURES))
def test_plan_json_is_byte_identical_to_reference_and_cross_loads(tag):
    """serialize_plan / parse_plan (placement.cpp:603-658): a plan the
    reference wrote loads here and is written back byte for byte, and the
    reference loads this engine's text back to the same bytes."""
    d = golden_cluster(ROUTE_FIXTURES[tag])
    text = ref_plan_json(d, golden(f"{tag}.npz")["row"])
    p = h.Plan.from_json(text)
    assert p.to_json() == text
    again = _text(_lib().refh_plan_roundtrip, p.to_json().encode())
    assert again == text
    z = golden(f"{tag}.npz")
    assert [e[2] for e in p.edges] == list(z["plan_flow"])
    assert p.objective == float(z["objective"][0])


@needs_ref
def test_plan_json_numbers_and_text_survive_both_ways():
    plan = {"method": "milp", "status": "feasible", "objective": 1e-05, "best_bound": 123456789012345.67,
            "allow_partial": False, "nodes_explored": 17,
            "nodes": [{"id": "nødé-α", "start": 0, "end": 3}],
            "edges": [{"src": "coord", "dst": "nødé-α", "flow": 0.30000000000000004, "exec_start": 0,
                       "exec_end": 3},
                      {"src": "nødé-α", "dst": "coord", "flow": 2.5e-300, "exec_start": 3, "exec_end": 3}]}
    text = _text(_lib().refh_plan_roundtrip, json.dumps(plan).encode())
    assert h.Plan.from_json(text).to_json() == text


@needs_ref
@pytest.mark.parametrize("name", ["het42-70b", "geo24", "syn256-120l"])
def test_cluster_json_is_byte_identical_to_reference(name):
    d = clusters.CONFIGS[name]("float")
    rc = RefCluster(d)
    lib = _lib()
    removed = C.c_int(0)
    # serialize_cluster of the reference's own parse (degree 1e9 prunes nothing)
    text = _text(lambda b, n: lib.refh_prune_json(rc.h, 1e9, b, n, C.byref(removed)))
    assert removed.value == 0
    assert h.Cluster.from_json(text).to_json() == text


@needs_ref
@needs_planner
def test_prune_links_het42_matches_reference():
    """the het42 prune_links(c, 12) variant."""
    d = clusters.CONFIGS["het42-70b"]("float")
    rc = RefCluster(d)
    removed = C.c_int(0)
    want = _text(lambda b, n: _lib().refh_prune_json(rc.h, 12.0, b, n, C.byref(removed)))
    pruned, rep = h.prune_links(_cluster(d), 12)
    assert pruned.to_json() == want
    assert rep["links_removed"] == removed.value == 1806 - pruned.num_links
    assert rep["avg_degree_after"] <= 12.0 + 1e-9
    assert json.loads(want) == clusters.CONFIGS["het42-70b-prune12"]("float")


@needs_planner
def test_upper_bound_and_policy_validation():
    d = golden_cluster("fan3")
    c = _cluster(d)
    assert h.throughput_upper_bound(c) > 0
    if not ref_available():
        return
    text = ref_plan_json(d, golden("route_fan3.npz")["row"])
    p = h.Plan.from_json(text)
    for pol in ("random", "sqf", "swarm"):
        with pytest.raises(h.ValidationError, match="iwrr only"):
            h.Scheduler(c, p, pol, 1)
    with pytest.raises(h.ValidationError, match="unknown scheduler policy"):
        h.Scheduler(c, p, "fifo", 1)


def test_generate_trace_returns_reference_tuples():
    t = h.generate_trace(5, 2.0, "online", 3)
    arr, i, o = ref_trace(5, 3, rate=2.0, online=True) if ref_available() else h.generate_trace_arrays(5, 2.0,
                                                                                                         "online", 3)
    assert t == [(float(a), int(x), int(y)) for a, x, y in zip(arr, i, o)]
    assert all(isinstance(x, tuple) and len(x) == 3 for x in t)


# --- GPU: stateful scheduler, simulator, MILP, plan edges, DOT -------------------

def _ops(rng, R, in_len, out_len, p_complete=0.45):
    """A random admit/complete interleaving over R requests (ids 0..R-1 in
    order; completes pick a random outstanding admitted id)."""
    kind, ids, lens = [], [], []
    outstanding = []
    nxt = 0
    while nxt < R or outstanding:
        if nxt < R and (not outstanding or rng.random() > p_complete):
            kind.append(0)
            ids.append(nxt)
            lens.append(int(in_len[nxt]))
            outstanding.append(nxt)
            nxt += 1
        else:
            j = outstanding.pop(int(rng.integers(len(outstanding))))
            kind.append(1)
            ids.append(j)
            lens.append(int(out_len[j]))
    return np.array(kind, np.int32), np.array(ids, np.int64), np.array(lens, np.int32)


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(ROUTE_FIXTURES))
def test_scheduler_interleaved_admit_complete_matches_reference(tag):
    """Scheduler(c, plan, iwrr, seed) with admits and completes interleaved
    the way the simulator drives it (sim.cpp:179-192, :225): routes, deferrals,
    per-node KV estimates and the running output mean identical, op by op.
    Completes of deferred ids are skipped on both sides (the simulator only
    completes admitted requests)."""
    d = golden_cluster(ROUTE_FIXTURES[tag])
    z = golden(f"{tag}.npz")
    row = np.ascontiguousarray(z["row"], np.int16)
    c = _cluster(d)
    text = ref_plan_json(d, row)
    plan = h.Plan.from_json(text)
    rng = np.random.default_rng(11)
    R = 3000
    kind, ids, lens = _ops(rng, R, z["in_len"][:R], z["out_len"][:R], 0.2 if tag == "route_kvmask" else 0.45)
    probe = next(e[1] for e in plan.edges if e[0] == d["coordinator"]["id"])
    K, H = len(kind), int(d["model"]["num_layers"])
    # the reference (completes of deferred ids are skipped on both sides)
    rc = RefCluster(d)
    nh = np.zeros(K, np.int32)
    hn = np.full(K * H, -9, np.int32)
    hs = np.zeros(K * H, np.int32)
    he = np.zeros(K * H, np.int32)
    kv = np.zeros(K, np.float64)
    avg = np.zeros(K, np.float64)
    err = C.create_string_buffer(512)
    assert _lib().refh_sched_ops(rc.h, row, 1, 7, K, kind, ids, lens, H, nh, hn, hs, he, probe.encode(), kv, avg,
                                 err, 512) == 0, err.value
    # this engine
    s = h.Scheduler(c, plan, "iwrr", 7)
    nid = {n["id"]: k for k, n in enumerate(d["nodes"])}
    n_def = 0
    deferred = set()
    for k in range(K):
        if kind[k] == 0:
            r = s.admit(int(ids[k]), int(lens[k]))
            if r is None:
                assert nh[k] == -1, k
                n_def += 1
                deferred.add(int(ids[k]))
            else:
                assert len(r) == nh[k], k
                for j, (node, a, b) in enumerate(r):
                    assert (nid[node], a, b) == (hn[k * H + j], hs[k * H + j], he[k * H + j]), (k, j)
        elif int(ids[k]) in deferred:
            assert nh[k] == -2, k
        else:
            s.complete(int(ids[k]), int(lens[k]))
        assert bits([s.kv_estimate(probe)])[0] == bits(kv[k : k + 1])[0], k
        assert bits([s.avg_output])[0] == bits(avg[k : k + 1])[0], k
    assert s.kv_capacity(probe) > 0
    if tag == "route_kvmask":
        assert n_def > 0  # the KV watermark binds on this plan


@needs_ref
@needs_planner
@pytest.mark.gpu
@pytest.mark.parametrize("name,online,n,rate,horizon", [("geo24", 0, 300, 0.0, 600.0), ("geo24", 1, 300, 0.5, 600.0),
                                                         ("fan3", 1, 600, 2.0, 300.0), ("kvmask", 1, 300, 0.5, 600.0),
                                                         ("kvmask", 0, 300, 0.0, 600.0)])
def test_simulate_matches_reference(name, online, n, rate, horizon):
    """simulate(c, plan, trace, scheduler="iwrr") — the reference's DES
    (sim.cpp) over this engine's Scheduler — reports the pure reference's
    metrics exactly (every key, every double bit), light and overloaded
    traces (millions of deferred re-admissions), KV-masked plan included."""
    tag = {"geo24": "route_geo24", "fan3": "route_fan3", "kvmask": "route_kvmask"}[name]
    d = golden_cluster(ROUTE_FIXTURES[tag])
    row = np.ascontiguousarray(golden(f"{tag}.npz")["row"], np.int16)
    arr, i, o = ref_trace(n, 5, rate=rate, online=bool(online))
    rc = RefCluster(d)
    want = json.loads(_text(_lib().refh_simulate, rc.h, row, 1, n, arr, i, o, online, 0, 3, horizon, 5.0))
    c = _cluster(d)
    plan = h.Plan.from_json(ref_plan_json(d, row))
    got = h.simulate(c, plan, [(float(a), int(x), int(y)) for a, x, y in zip(arr, i, o)],
                     "online" if online else "offline", "iwrr", 3, horizon, 5.0)
    assert got == want
    assert got["requests_completed_total"] > 0


@needs_ref
@needs_planner
@pytest.mark.gpu
def test_plan_milp_through_the_product_matches_pure_reference():
    """plan(c, "milp") — the reference's plan_placement linked over this
    engine — takes the pure reference's branch-and-bound path exactly
    (objective bits, placement, status, bound, explored nodes) on the AC2
    clusters of the search fixture (both modes) and the reference's default
    options otherwise."""
    from _support import plan_milp
    z = golden("search_exhaustive.npz")
    lib = ref()
    for i, key in enumerate(z["keys"][:24]):
        d = golden_cluster(str(key))
        N = len(d["nodes"])
        p = bool(z["partial"][i])
        rc = RefCluster(d)
        obj, row, st, bb, nodes = plan_milp(lib, "refh_", rc.h, N, p, gap=0.0, lex=False)
        got = h.plan(_cluster(d), "milp", allow_partial=p, gap=0.0, lex_tiebreak=False)
        assert bits([got.objective])[0] == bits([obj])[0], key
        assert got.placement == _placement(d, row), key
        assert bits([got.best_bound])[0] == bits([bb])[0], key
        assert got.optimal == (st == 0), key
        assert got.method == "milp"


@needs_ref
@pytest.mark.gpu
def test_plan_edges_match_reference_plan_from_placement():
    """plan_for_placement's edges (src, dst, flow bits, exec range) equal the
    reference's plan_from_placement (placement.cpp:440-469) on the route
    fixtures and on sampled candidate rows of every config."""
    cases = [(ROUTE_FIXTURES[t], golden(f"{t}.npz")["row"]) for t in sorted(ROUTE_FIXTURES)]
    for key in ("het42-70b_float", "geo24_float", "single24-30b_int", "syn256-120l_float"):
        rows = golden(f"cand_{key}.npz")["rows"]
        st = golden(f"cand_{key}.npz")["status_partial"]
        ok = np.nonzero(st == 0)[0]
        for j in ok[:: max(1, len(ok) // 12)][:12]:
            cases.append((key, rows[j]))
    for key, row in cases:
        d = golden_cluster(key)
        want = h.Plan.from_json(ref_plan_json(d, row))
        got = h.plan_for_placement(_cluster(d), _placement(d, row))
        assert got.edges == want.edges, key
        assert bits([got.objective])[0] == bits([want.objective])[0], key
        assert got.to_json() == want.to_json()


@needs_ref
@pytest.mark.gpu
def test_to_dot_and_min_cut_match_reference():
    """to_dot (flow_graph.cpp:257-271) byte for byte and min_cut_source_side
    (:231-255) after this engine's max_flow."""
    lib = _lib()
    for key in ("geo24_float", "het42-70b_float", "fan3"):
        d = golden_cluster(key)
        rows = golden("route_fan3.npz")["row"][None] if key == "fan3" else golden(f"cand_{key}.npz")["rows"][:6]
        rc = RefCluster(d)
        c = _cluster(d)
        for row in rows:
            row = np.ascontiguousarray(row, np.int16)
            cut = np.zeros(4 * len(d["nodes"]) + 4, np.int32)
            ncut = C.c_int(0)
            buf = C.create_string_buffer(1 << 20)
            n = lib.refh_to_dot(rc.h, row, 1, buf, 1 << 20, cut, C.byref(ncut))
            if n < 0:
                continue  # invalid row: the reference throws; build_flow_graph below must too
            g = h.build_flow_graph(c, _placement(d, row))
            h.max_flow(g)
            assert g.to_dot() == buf.value.decode(), key
            assert list(g.min_cut_source_side()) == list(cut[: ncut.value]), key
