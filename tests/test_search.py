"""Placement search: the reference's baseline
heuristics (src/heuristics.cpp:12-131) restated on the host as local-search
seeds, and the device best-improvement local search checked move for move
against the same driver run over the reference's own scorer."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters

from _support import RefCluster, local_search_oracle, ref, ref_available, ref_heuristic

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
METHODS = ("swarm", "petals", "sp")


def _cluster(d):
    return h.Cluster.from_json(json.dumps(d))


def _row(c, placement):
    return h.placement_rows(c, [{k: tuple(v) for k, v in placement.items()}])[0]


def _random_cluster(seed, max_nodes=10, lo=4, hi=10):
    # random_cluster.hpp loops forever unless 2 * (max_hold + 2) >= L: keep L <= 10
    lib = ref()
    lib.refh_random_cluster_json.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]
    lib.refh_random_cluster_json.restype = C.c_int
    buf = C.create_string_buffer(1 << 16)
    n = lib.refh_random_cluster_json(seed, max_nodes, lo, hi, buf, 1 << 16)
    assert n > 0
    return json.loads(buf.value.decode())


# --- heuristics (host; no GPU) ------------------------------------------------

@needs_ref
@pytest.mark.parametrize("name", ["het42-70b", "geo24", "single24-30b", "single24-70b", "syn256-120l"])
@pytest.mark.parametrize("method", METHODS)
def test_heuristic_matches_reference(name, method):
    d = clusters.CONFIGS[name]()
    c = _cluster(d)
    want_row, want_warn = ref_heuristic(RefCluster(d), method)
    placement, warnings = h.heuristic_placement(c, method)
    assert np.array_equal(_row(c, placement), want_row)
    assert warnings == want_warn


@needs_ref
def test_heuristics_match_reference_on_random_clusters():
    checked = 0
    for seed in range(60):
        d = _random_cluster(9100 + seed)
        c = _cluster(d)
        rc = RefCluster(d)
        for method in METHODS:
            want_row, want_warn = ref_heuristic(rc, method)
            placement, warnings = h.heuristic_placement(c, method)
            assert np.array_equal(_row(c, placement), want_row), (seed, method)
            assert warnings == want_warn, (seed, method)
            checked += 1
    assert checked == 180


@needs_ref
def test_separate_pipelines_needs_types():
    d = clusters.CONFIGS["geo24"]()
    d["nodes"][3]["type"] = ""
    with pytest.raises(ValueError) as want:
        ref_heuristic(RefCluster(d), "sp")
    with pytest.raises(h.ValidationError) as got:
        h.heuristic_placement(_cluster(d), "sp")
    assert str(got.value) == str(want.value)


def test_neighbour_order_is_enumerate_choice_order():
    from _support import neighbour_moves

    node, s, e, pa = neighbour_moves([1, 2], 3)
    got = list(zip(node.tolist(), s.tolist(), e.tolist()))
    assert got == [(0, 0, 0), (0, 0, 1), (0, 1, 2), (0, 2, 3),
                   (1, 0, 0), (1, 0, 1), (1, 0, 2), (1, 1, 2), (1, 1, 3), (1, 2, 3)]
    assert (pa == -1).all()
    node, s, e, pa = neighbour_moves([1, 2, 1], 3, swaps=True)
    assert list(zip(node[pa >= 0].tolist(), pa[pa >= 0].tolist())) == [(0, 1), (0, 2), (1, 2)]


# --- device local search ------------------------------------------------------

def _ref_scorer(d, partial=True):
    rc = RefCluster(d)
    threads = os.cpu_count() or 1
    return rc, (lambda rows: rc.score(rows, partial, threads))


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name,seed_method,max_moves,swaps", [
    ("geo24", "petals", -1, True), ("geo24", "swarm", -1, False), ("geo24", "swarm", -1, True),
    ("single24-30b", "petals", -1, True), ("het42-70b", "petals", 2, True),
])
def test_local_search_matches_reference_driver(name, seed_method, max_moves, swaps):
    d = clusters.CONFIGS[name]()
    c = _cluster(d)
    seed = _row(c, h.heuristic_placement(c, seed_method)[0])
    e = h.Engine(c)  # PARITY: every value is the reference's double
    value, row, moves, scored = e.local_search(seed, True, max_moves, swaps)
    rc, score = _ref_scorer(d)
    w_value, w_row, w_moves, w_scored = local_search_oracle(score, list(e.kmax), rc.L, seed, max_moves, swaps)
    assert value == w_value
    assert np.array_equal(row, w_row)
    assert (moves, scored) == (w_moves, w_scored)
    if max_moves < 0:
        assert moves > 0


@pytest.mark.gpu
def test_local_search_score_mode_integer_capacities_equal_parity():
    d = clusters.CONFIGS["het42-70b"]("int")
    c = _cluster(d)
    seed = _row(c, h.heuristic_placement(c, "swarm")[0])
    e = h.Engine(c)
    par = e.local_search(seed, True, 4)
    e.mode = "score"
    sco = e.local_search(seed, True, 4)
    assert par[0] == sco[0] and np.array_equal(par[1], sco[1]) and par[2:] == sco[2:]


@pytest.mark.gpu
def test_local_search_is_a_local_optimum():
    d = clusters.CONFIGS["geo24"]()
    c = _cluster(d)
    e = h.Engine(c)
    seed = _row(c, h.heuristic_placement(c, "swarm")[0])
    value, row, moves, scored = e.local_search(seed)
    again = e.local_search(row)
    assert again[0] == value and again[2] == 0 and np.array_equal(again[1], row)
    # and the value is the device's PARITY value of the final row
    v, st = e.score(row[None])
    assert st[0] == 0 and v[0] == value


@pytest.mark.gpu
def test_plan_local_beats_its_seeds():
    d = clusters.CONFIGS["geo24"]()
    c = _cluster(d)
    p = h.plan(c, "local")
    assert p.method == "local"
    for m in METHODS:
        assert p.objective >= h.plan(c, m).objective
    assert p.objective == h.max_flow_value(c, p.placement)
    # the best seed's local optimum, via the module-level entry
    best = max((h.local_search(c, h.heuristic_placement(c, m)[0])[1] for m in METHODS))
    assert p.objective == best


@pytest.mark.gpu
def test_plan_sampled_at_least_local():
    """plan(c, "sampled"): each seed's local optimum, then the sampled
    multi-node search, then local search again; never below plan(c, "local"),
    deterministic, and its objective is the reference-exact max-flow value."""
    for name in ("geo24", "geo24-70b"):
        c = _cluster(clusters.CONFIGS[name]())
        p = h.plan(c, "sampled")
        assert p.method == "sampled"
        assert p.objective >= h.plan(c, "local").objective
        assert p.objective == h.max_flow_value(c, p.placement)
        assert h.plan(c, "sampled").objective == p.objective


@pytest.mark.gpu
def test_plan_search_on_syn256_scores_moves_in_score_mode_and_returns_parity_values():
    """Clusters above 64 nodes score search moves in SCORE mode and re-solve
    the result in PARITY (shim_heuristics.cpp): the objective is the
    reference-exact max-flow of the returned placement and never below a seed."""
    c = _cluster(clusters.CONFIGS["syn256-120l"]())
    seeds = {m: h.plan(c, m).objective for m in ("swarm", "petals")}
    p = h.plan(c, "local")
    assert p.objective == h.max_flow_value(c, p.placement)
    assert all(p.objective >= v for v in seeds.values())
    q = h.plan(c, "sampled")
    assert q.objective == h.max_flow_value(c, q.placement)
    assert q.objective >= p.objective


@pytest.mark.gpu
def test_local_search_rejects_invalid_seed():
    d = clusters.CONFIGS["geo24"]()
    c = _cluster(d)
    e = h.Engine(c)
    bad = np.zeros((len(d["nodes"]), 2), np.int16)
    bad[0] = (0, 24)  # longer than node 0's VRAM allows
    with pytest.raises(Exception):
        e.local_search(bad)
    with pytest.raises(h.ValidationError):
        h.local_search(c, {d["nodes"][0]["id"]: (0, 24)})


@pytest.mark.gpu
@needs_ref
def test_sampled_search_escapes_the_local_optimum():
    """helio_gpu_sampled_search: multi-node mutants of the incumbent, first
    strict best kept.  From geo24's swarm seed the single-node local optimum
    (866.7) is left behind; the result is reproducible, never below its seed,
    and its PARITY value is the reference's value of the returned row."""
    d = clusters.CONFIGS["geo24"]()
    c = _cluster(d)
    e = h.Engine(c)  # PARITY
    seed = _row(c, h.heuristic_placement(c, "swarm")[0])
    lv, lrow, _, _ = e.local_search(seed)
    v1, r1, imp, scored = e.sampled_search(lrow, True, 8, 200_000, 3, 7)
    v2, r2, imp2, scored2 = e.sampled_search(lrow, True, 8, 200_000, 3, 7)
    assert v1 == v2 and np.array_equal(r1, r2) and (imp, scored) == (imp2, scored2)
    assert scored == 1 + 8 * 200_000
    assert v1 > lv and imp >= 1
    rc, score = _ref_scorer(d)
    ref_v, ref_st = score(np.ascontiguousarray(r1[None]))
    assert ref_st[0] == 0 and ref_v[0] == v1
    # zero rounds return the seed untouched
    v0, r0, imp0, sc0 = e.sampled_search(lrow, True, 0, 1000, 3, 7)
    assert v0 == lv and np.array_equal(r0, lrow) and imp0 == 0 and sc0 == 1


@pytest.mark.gpu
def test_sampled_search_score_mode_integer_capacities_equal_parity():
    d = clusters.CONFIGS["het42-70b"]("int")
    c = _cluster(d)
    e = h.Engine(c)
    seed = _row(c, h.heuristic_placement(c, "petals")[0])
    par = e.sampled_search(seed, True, 3, 100_000, 2, 11)
    e.mode = "score"
    sco = e.sampled_search(seed, True, 3, 100_000, 2, 11)
    assert par[0] == sco[0] and np.array_equal(par[1], sco[1]) and par[2:] == sco[2:]
