"""CPU: pin the C oracle (oracle/helio_oracle.c) against the golden vectors
generated from the compiled reference (tests/golden/make_golden.py), and check
that the candidate generator's host copy matches the fixture generator."""

import numpy as np
import pytest

from _support import (CAND_FIXTURES, Oracle, bits, golden, golden_cluster, iwrr_weights_oracle,
                      max_flow_raw_oracle)


@pytest.mark.parametrize("kind", ["ac1", "testflow"])
def test_raw_graphs_match_reference(kind):
    g = golden(f"raw_{kind}.npz")
    G = len(g["n"])
    for i in range(G):
        a, b = g["off"][i], g["off"][i + 1]
        val, flow = max_flow_raw_oracle(int(g["n"][i]), int(g["s"][i]), int(g["t"][i]),
                                        g["u"][a:b], g["v"][a:b], g["cap"][a:b])
        assert bits([val])[0] == bits(g["values"][i : i + 1])[0], (kind, i)
        assert np.array_equal(bits(flow), bits(g["flows"][a:b])), (kind, i)


def test_ac1_values_are_integers_and_match_edmonds_karp_count():
    # AC1 asserts exact == against Edmonds-Karp; the reference's own values
    # are integral, so the fixture must be too.
    g = golden("raw_ac1.npz")
    assert np.all(g["values"] == np.round(g["values"]))
    assert len(g["n"]) == 1000


@pytest.mark.parametrize("key", CAND_FIXTURES)
def test_candidates_match_reference(key):
    z = golden(f"cand_{key}.npz")
    o = Oracle(golden_cluster(key))
    assert o.kmax() == list(z["kmax"])
    for partial, vk, sk in ((True, "values_partial", "status_partial"),
                            (False, "values_strict", "status_strict")):
        v, s = o.score(z["rows"], partial)
        assert np.array_equal(s, z[sk]), key
        assert np.array_equal(bits(v), bits(z[vk])), key
    for b in range(len(z["graph_ne"])):
        st, nv, edges, val = o.graph(z["rows"][b], True)
        if z["status_partial"][b] != 0:
            assert st == z["status_partial"][b]
            continue
        ne = int(z["graph_ne"][b])
        assert nv == z["graph_nv"][b] and len(edges["u"]) == ne
        gi, gd = z["graph_ints"][b, :ne], z["graph_dbl"][b, :ne]
        for j, k in enumerate(("u", "v", "kind", "es", "ee")):
            assert np.array_equal(edges[k], gi[:, j]), (key, b, k)
        assert np.array_equal(bits(edges["cap"]), bits(gd[:, 0])), (key, b)
        assert np.array_equal(bits(edges["flow"]), bits(gd[:, 1])), (key, b)
        assert bits([val])[0] == bits(z["graph_value"][b : b + 1])[0]


@pytest.mark.parametrize("tag", ["geo24", "fan3", "kvmask"])
def test_routes_match_reference(tag):
    z = golden(f"route_{tag}.npz")
    o = Oracle(golden_cluster({"geo24": "geo24_float"}.get(tag, tag)))
    n, pe, obj = o.plan(z["row"])
    assert n == len(z["plan_src"]) and obj == z["objective"][0]
    for k, gk in (("src", "plan_src"), ("dst", "plan_dst"), ("es", "plan_es"), ("ee", "plan_ee")):
        assert np.array_equal(pe[k], z[gk])
    assert np.array_equal(bits(pe["flow"]), bits(z["plan_flow"]))
    den, nh, hn, hs, he = o.route(z["row"], z["in_len"], z["out_len"])
    assert den == z["deferred"][0]
    assert np.array_equal(nh, z["nh"])
    H = hn.shape[1]
    mask = np.arange(H)[None, :] < np.maximum(nh, 0)[:, None]
    for a, b in ((hn, z["hop_node"]), (hs, z["hop_s"]), (he, z["hop_e"])):
        assert np.array_equal(a[mask], b[mask])


def test_iwrr_weights_match_reference():
    z = golden("iwrr.npz")
    off = z["flows_off"]
    for i in range(len(off) - 1):
        a, b = off[i], off[i + 1]
        assert np.array_equal(iwrr_weights_oracle(z["flows"][a:b]), z["weights"][a:b])
    # test_scheduler.cpp:62-68 known answers
    assert list(iwrr_weights_oracle([2.0, 1.0])) == [32, 16]
    assert list(iwrr_weights_oracle([1000.0, 381.47])) == [32, 12]
    assert list(iwrr_weights_oracle([0.0001])) == [1]
    assert list(iwrr_weights_oracle([0.002, 0.001])) == [2, 1]
    assert list(iwrr_weights_oracle([5.0, 0.0001])) == [32, 1]


def test_fan3_ac8_split_within_tolerance():
    # AC8 (acceptance_main.cpp:505-553): weights 32:19:13, 10k admissions,
    # per-replica counts within 3 of 10000 * w / sum(w).
    z = golden("route_fan3.npz")
    w = iwrr_weights_oracle(z["plan_flow"][z["plan_src"] == -1])
    assert list(w) == [32, 19, 13]
    counts = np.bincount(z["hop_node"][:, 0], minlength=3)
    expect = 10000 * w / w.sum()
    assert np.all(np.abs(counts - expect) <= 3)


def test_host_generator_matches_fixture_generator():
    from paper_2406_01566_b200 import generate_host
    import importlib.util, os
    spec = importlib.util.spec_from_file_location(
        "make_golden", os.path.join(os.path.dirname(__file__), "golden", "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    for key in ("het42-70b_float", "geo24_float", "single24-30b_float"):
        z = golden(f"cand_{key}.npz")
        k = [int(x) for x in z["kmax"]]
        L = golden_cluster(key)["model"]["num_layers"]
        seed = int(z["seed"][0])
        for first, ppm in ((0, 0), (1000, 200000)):
            a = generate_host(k, L, seed, first, 16, ppm)
            b = mg.kgen(len(k), L, k, seed, first, 16, ppm)
            assert np.array_equal(a, b)
        n0 = len(z["rows"]) - 0
        assert np.array_equal(generate_host(k, L, seed, 0, 8, 0), z["rows"][:8])


@pytest.mark.parametrize("config", ["het42-70b", "single24-30b", "geo24"])
def test_reference_arm_generator_matches_product_generator(config):
    """bench.py --impl reference draws its rows with refh_generate (over the
    reference's ClusterSpec) so it loads nothing from the package: the rows must
    be the product generator's (csrc/gen.h) exactly, chains and uniform mixes."""
    from paper_2406_01566_b200 import clusters, generate_host
    from _support import RefCluster, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = clusters.CONFIGS[config]("float")
    rc = RefCluster(d)
    k = [int(rc.lib.refh_max_layers(rc.h, i)) for i in range(rc.N)]
    L = int(d["model"]["num_layers"])
    for first, ppm, threads in ((0, 0, 1), (123456, 100000, 4), (10**9, 0, 3)):
        a = generate_host(k, L, 20240611, first, 257, ppm)
        b = rc.generate(20240611, first, 257, ppm, False, threads)
        assert np.array_equal(a, b)
