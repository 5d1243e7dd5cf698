"""GPU parity: the CUDA path (through the C ABI, via the _helio bindings)
against the golden vectors from the compiled reference and against the C
oracle on seeded inputs.  Integer/index results must be identical; doubles
must be BIT-identical (PARITY semantics replay the reference's FIFO discharge,
so no tolerance is needed even for float capacities — north_star allows
1e-6 relative for float capacities; we assert 0 ulp)."""

import json

import numpy as np
import pytest

import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
from _support import CAND_FIXTURES, Oracle, bits, golden, golden_cluster

pytestmark = pytest.mark.gpu

_engines = {}


def engine(key):
    if key not in _engines:
        c = h.Cluster.from_json(json.dumps(golden_cluster(key)))
        _engines[key] = (c, h.Engine(c))
    return _engines[key]


def test_engine_is_native():
    c, e = engine("geo24_float")
    assert e.launch_count >= 0
    import os
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libhelio_gpu.so" in maps


@pytest.mark.parametrize("kind", ["ac1", "testflow"])
def test_raw_graphs_bit_exact(kind):
    g = golden(f"raw_{kind}.npz")
    vals, flows = h.max_flow_raw(g["n"], g["s"], g["t"], g["off"], g["u"], g["v"], g["cap"])
    assert np.array_equal(bits(vals), bits(g["values"]))
    assert np.array_equal(bits(flows), bits(g["flows"]))


@pytest.mark.parametrize("key", CAND_FIXTURES)
def test_candidate_values_bit_exact(key):
    z = golden(f"cand_{key}.npz")
    c, e = engine(key)
    assert list(e.kmax) == list(z["kmax"])
    for partial, vk, sk in ((True, "values_partial", "status_partial"),
                            (False, "values_strict", "status_strict")):
        v, s = e.score(z["rows"], partial)
        assert np.array_equal(s, z[sk]), key
        assert np.array_equal(bits(v), bits(z[vk])), key


@pytest.mark.parametrize("key", CAND_FIXTURES)
def test_candidate_graphs_and_flows_bit_exact(key):
    z = golden(f"cand_{key}.npz")
    c, e = engine(key)
    G = len(z["graph_ne"])
    vals, st, nv, ne, ints, dbl = e.flows(z["rows"][:G], True)
    assert np.array_equal(st, z["status_partial"][:G])
    for b in range(G):
        if st[b] != 0:
            continue
        n = int(z["graph_ne"][b])
        assert nv[b] == z["graph_nv"][b] and ne[b] == n
        assert np.array_equal(ints[b, :n, :5], z["graph_ints"][b, :n]), (key, b)
        assert np.array_equal(bits(dbl[b, :n, 0]), bits(z["graph_dbl"][b, :n, 0])), (key, b)
        assert np.array_equal(bits(dbl[b, :n, 1]), bits(z["graph_dbl"][b, :n, 1])), (key, b)
        assert bits(vals[b : b + 1])[0] == bits(z["graph_value"][b : b + 1])[0]


@pytest.mark.parametrize("name", ["het42-70b", "single24-30b", "geo24", "geo24-70b"])
@pytest.mark.parametrize("cap", ["float", "int"])
def test_seeded_batches_match_oracle(name, cap):
    d = clusters.CONFIGS[name](cap)
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    o = Oracle(d)
    k = list(e.kmax)
    assert k == o.kmax()
    rows = np.concatenate([h.generate_host(k, c.num_layers, 77, 0, 1500, 0),
                           h.generate_host(k, c.num_layers, 77, 10**6, 500, 150000)])
    for partial in (True, False):
        v, s = e.score(rows, partial)
        vo, so = o.score(rows, partial)
        assert np.array_equal(s, so)
        assert np.array_equal(bits(v), bits(vo))


def test_syn256_overflow_path_matches_oracle():
    # 256 nodes, V = 514: exercises the large-slot (one warp per CTA) path.
    d = clusters.CONFIGS["syn256-120l"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    o = Oracle(d)
    rows = h.generate_host(list(e.kmax), c.num_layers, 5, 0, 64, 300000)
    v, s = e.score(rows)
    vo, so = o.score(rows)
    assert np.array_equal(s, so) and np.array_equal(bits(v), bits(vo))


def test_device_generator_matches_host():
    import torch
    c, e = engine("het42-70b_float")
    B = 100_000
    out = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda")
    e.generate_device(123, 5_000_000, B, 100000, out.data_ptr(), 0)
    torch.cuda.synchronize()
    host = h.generate_host(list(e.kmax), c.num_layers, 123, 5_000_000, B, 100000)
    assert np.array_equal(out.cpu().numpy(), host)


def test_device_scoring_and_argmax():
    import torch
    c, e = engine("het42-70b_float")
    B = 50_000
    pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda")
    e.generate_device(9, 0, B, 50000, pl.data_ptr(), 0)
    vals = torch.empty(B, dtype=torch.float64, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    e.score_device(pl.data_ptr(), B, vals.data_ptr(), st.data_ptr(), True, 0)
    best = torch.empty(1, dtype=torch.float64, device="cuda")
    idx = torch.empty(1, dtype=torch.int64, device="cuda")
    e.argmax_device(vals.data_ptr(), st.data_ptr(), B, 1000, best.data_ptr(), idx.data_ptr(), 0)
    torch.cuda.synchronize()
    v = vals.cpu().numpy()
    s = st.cpu().numpy()
    hv, hs = e.score(pl.cpu().numpy())
    assert np.array_equal(bits(v), bits(hv)) and np.array_equal(s, hs)
    ok = (s == 0) & (v > 0)
    i = int(np.argmax(np.where(ok, v, -1.0)))
    assert int(idx.item()) == i + 1000 and best.item() == v[i]
    # spot-check against the oracle
    o = Oracle(golden_cluster("het42-70b_float"))
    sub = np.random.default_rng(0).choice(B, 400, replace=False)
    vo, so = o.score(pl.cpu().numpy()[sub])
    assert np.array_equal(bits(v[sub]), bits(vo))


def test_scoring_is_deterministic_at_full_size():
    # SURVEY §8(d) headline size: 1M het42 candidates; size-independent
    # properties: repeat-run identity, status all OK, values > 0 for chains,
    # and a seeded subsample bit-exact against the oracle.
    import torch
    c, e = engine("het42-70b_float")
    B = 1_000_000
    pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda")
    e.generate_device(2024, 0, B, 0, pl.data_ptr(), 0)
    v1 = torch.empty(B, dtype=torch.float64, device="cuda")
    v2 = torch.empty(B, dtype=torch.float64, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    e.score_device(pl.data_ptr(), B, v1.data_ptr(), st.data_ptr(), True, 0)
    e.score_device(pl.data_ptr(), B, v2.data_ptr(), st.data_ptr(), True, 0)
    torch.cuda.synchronize()
    assert torch.equal(v1.view(torch.int64), v2.view(torch.int64))
    assert int((st != 0).sum()) == 0
    o = Oracle(golden_cluster("het42-70b_float"))
    sub = np.random.default_rng(1).choice(B, 1000, replace=False)
    vo, so = o.score(pl.cpu().numpy()[sub])
    assert np.array_equal(bits(v1.cpu().numpy()[sub]), bits(vo))


@pytest.mark.parametrize("cap", ["int", "float"])
def test_syn256_at_scale_is_deterministic_and_matches_the_reference(cap):
    """configs[4] at scale: 1M syn256 link walks in SCORE mode (the large-graph
    kernel, all slot tiers) — repeat-run identity, every status OK, the argmax
    equal to the first maximum of the returned values, and a seeded subsample
    against the reference's own build_flow_graph + max_flow (bit-exact on
    integer capacities, 1e-6 relative on float)."""
    import torch
    from _support import RefCluster, ref_available
    d = clusters.CONFIGS["syn256-120l"](cap)
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    e.mode = "score"
    B = 1_000_000
    pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda")
    e.generate_walk_device(99, 0, B, pl.data_ptr(), 0)
    v1 = torch.empty(B, dtype=torch.float64, device="cuda")
    v2 = torch.empty(B, dtype=torch.float64, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    best = torch.empty(1, dtype=torch.float64, device="cuda")
    idx = torch.empty(1, dtype=torch.int64, device="cuda")
    e.score_device(pl.data_ptr(), B, v1.data_ptr(), st.data_ptr(), True, 0)
    e.score_device(pl.data_ptr(), B, v2.data_ptr(), st.data_ptr(), True, 0)
    e.argmax_device(v1.data_ptr(), st.data_ptr(), B, 0, best.data_ptr(), idx.data_ptr(), 0)
    torch.cuda.synchronize()
    assert torch.equal(v1.view(torch.int64), v2.view(torch.int64))
    assert int((st != 0).sum()) == 0
    vh = v1.cpu().numpy()
    assert int(idx.item()) == int(np.argmax(vh)) and float(best.item()) == float(vh.max())
    sub = np.random.default_rng(2).choice(B, 300, replace=False)
    rows = pl.cpu().numpy()[sub]
    if ref_available():
        vo, so = RefCluster(d).score(rows, True, 8)
    else:
        vo, so = Oracle(d).score(rows)
    assert np.all(so == 0)
    if cap == "int":
        assert np.array_equal(bits(vh[sub]), bits(vo))
    else:
        assert np.all(np.abs(vh[sub] - vo) <= 1e-6 * np.maximum(1.0, np.abs(vo)))


@pytest.mark.parametrize("tag", ["geo24", "fan3", "kvmask"])
def test_routes_bit_exact(tag):
    z = golden(f"route_{tag}.npz")
    key = {"geo24": "geo24_float"}.get(tag, tag)
    c, e = engine(key)
    pe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
    nh, hn, hs, he, den = e.route(z["row"], pe, z["plan_flow"], z["in_len"], z["out_len"],
                                  z["hop_node"].shape[1])
    assert den == z["deferred"][0]
    assert np.array_equal(nh, z["nh"])
    mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
    for a, b in ((hn, z["hop_node"]), (hs, z["hop_s"]), (he, z["hop_e"])):
        assert np.array_equal(a[mask], b[mask])


def test_routes_one_million_match_oracle():
    z = golden("route_geo24.npz")
    c, e = engine("geo24_float")
    _, inl, outl = h.generate_trace_arrays(1_000_000, 0.0, "offline", 7)
    pe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
    nh, hn, hs, he, den = e.route(z["row"], pe, z["plan_flow"], inl, outl, c.num_layers)
    o = Oracle(golden_cluster("geo24_float"))
    den_o, nh_o, hn_o, hs_o, he_o = o.route(z["row"], inl, outl)
    assert den == den_o and np.array_equal(nh, nh_o)
    mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
    assert np.array_equal(hn[mask], hn_o[mask])
    assert np.array_equal(hs[mask], hs_o[mask]) and np.array_equal(he[mask], he_o[mask])


def test_masked_replay_division_is_ieee_division():
    """route.cu div_by_count (reciprocal computed ahead, then two FMAs) gives
    exactly a / n on 1e8 operand pairs of the routing domain (|a| < 2048,
    n < 2^27) — the running-mean update must be the reference's bits."""
    c, e = engine("geo24_float")
    assert e.check_division(100_000_000, 12345) == 0
    assert e.check_division(100_000_000, 777) == 0


@pytest.mark.parametrize("kv", [1e6, 7e5, 2e6])
def test_masked_routes_one_million_match_reference(kv):
    """KV masking binds (geo24's plan with kv_bytes_per_token_layer raised so
    13-96% of admissions are deferred): the exact replay (route_masked_spec)
    against the reference's Scheduler::admit/complete on 1M requests."""
    import copy
    from _support import RefCluster, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    z = golden("route_geo24.npz")
    d = copy.deepcopy(golden_cluster("geo24_float"))
    d["model"]["kv_bytes_per_token_layer"] = kv
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    _, inl, outl = h.generate_trace_arrays(1_000_000, 0.0, "offline", 7)
    pe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
    nh, hn, hs, he, den = e.route(z["row"], pe, z["plan_flow"], inl, outl, c.num_layers)
    den_r, nh_r, hn_r, hs_r, he_r = RefCluster(d).route(z["row"], inl, outl)
    assert 0 < den_r < 1_000_000
    assert den == den_r and np.array_equal(nh, nh_r)
    mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
    assert np.array_equal(hn[mask], hn_r[mask])
    assert np.array_equal(hs[mask], hs_r[mask]) and np.array_equal(he[mask], he_r[mask])


def _masked_case(kv, plan="golden"):
    import copy
    if plan == "golden":
        z = golden("route_geo24.npz")
        d = copy.deepcopy(golden_cluster("geo24_float"))
        row, pf = z["row"], z["plan_flow"]
        pe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
    else:  # bench.py routing_leg's plan: first max of 100k geo24 candidates
        import torch
        d = clusters.CONFIGS["geo24"]("float")
        c0 = h.Cluster.from_json(json.dumps(d))
        e0 = h.Engine(c0)
        e0.mode = "score"
        B = 100_000
        pl = torch.empty((B, e0.num_nodes, 2), dtype=torch.int16, device="cuda:0")
        sp = torch.cuda.current_stream().cuda_stream
        e0.generate_device(20240611, 0, B, 0, pl.data_ptr(), sp)
        v = torch.empty(B, dtype=torch.float64, device="cuda:0")
        st = torch.empty(B, dtype=torch.int32, device="cuda:0")
        bv = torch.empty(1, dtype=torch.float64, device="cuda:0")
        bi = torch.empty(1, dtype=torch.int64, device="cuda:0")
        e0.score_device(pl.data_ptr(), B, v.data_ptr(), st.data_ptr(), True, sp)
        e0.argmax_device(v.data_ptr(), st.data_ptr(), B, 0, bv.data_ptr(), bi.data_ptr(), sp)
        torch.cuda.synchronize()
        row = pl[int(bi.item())].cpu().numpy()
        pe, pf, _ = e0.plan_edges(row)
    d["model"]["kv_bytes_per_token_layer"] = kv
    return d, row, pe, pf


@pytest.mark.parametrize("variant", ["spec", "spec_exact_passes", "warp"])
@pytest.mark.parametrize("plan,kv", [("golden", 1e6), ("golden", 5e6), ("bench", 1e6), ("bench", 3e6)])
def test_masked_replay_variants_match_reference(variant, plan, kv, monkeypatch):
    """The three exact replays of route.cu on the same masked workloads, each
    against the reference's Scheduler::admit/complete: route_masked_spec
    (approximate first pass + verification), route_masked_spec with exact
    passes only (HELIO_ROUTE_APPROX=0: speculation on the deferral set with
    restarts), and the serial route_masked_warp (HELIO_ROUTE_SPEC=0).  bench
    is bench.py's routing plan (3% of 1M admissions deferred at kv 1e6)."""
    from _support import RefCluster, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    if variant == "spec_exact_passes":
        monkeypatch.setenv("HELIO_ROUTE_APPROX", "0")
    elif variant == "warp":
        monkeypatch.setenv("HELIO_ROUTE_SPEC", "0")
    d, row, pe, pf = _masked_case(kv, plan)
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    R = 1_000_000 if variant == "spec" else 300_000
    _, inl, outl = h.generate_trace_arrays(R, 0.0, "offline", 7)
    nh, hn, hs, he, den = e.route(row, pe, pf, inl, outl, c.num_layers)
    den_r, nh_r, hn_r, hs_r, he_r = RefCluster(d).route(row, inl, outl)
    assert 0 < den_r
    assert den == den_r and np.array_equal(nh, nh_r)
    mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
    assert np.array_equal(hn[mask], hn_r[mask])
    assert np.array_equal(hs[mask], hs_r[mask]) and np.array_equal(he[mask], he_r[mask])


def test_masked_replay_many_vertices_matches_reference():
    """A het42 plan (more routed vertices than the kernel has vertex warps, so
    warps own several vertices) under KV masking: route_masked_spec against
    the reference's Scheduler on 200k requests, for several kv sizes."""
    from _support import RefCluster, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    e.mode = "score"
    rows = h.generate_host(list(e.kmax), c.num_layers, 5, 0, 20_000, 20_000)
    v, st = e.score(rows)
    ok = (st == 0) & (v > 0)
    # the placement using the most nodes among the good ones
    used = (rows[:, :, 1] > rows[:, :, 0]).sum(1)
    cand = np.nonzero(ok & (v >= np.quantile(v[ok], 0.5)))[0]
    row = rows[cand[np.argmax(used[cand])]]
    pe, pf, _ = e.plan_edges(row)
    _, inl, outl = h.generate_trace_arrays(200_000, 0.0, "offline", 7)
    seen_partial = False
    for kv in (2e5, 1e6, 5e6):
        dm = json.loads(json.dumps(d))
        dm["model"]["kv_bytes_per_token_layer"] = kv
        cm = h.Cluster.from_json(json.dumps(dm))
        em = h.Engine(cm)
        nh, hn, hs, he, den = em.route(row, pe, pf, inl, outl, cm.num_layers)
        den_r, nh_r, hn_r, hs_r, he_r = RefCluster(dm).route(row, inl, outl)
        assert den == den_r and np.array_equal(nh, nh_r)
        mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
        assert np.array_equal(hn[mask], hn_r[mask])
        assert np.array_equal(hs[mask], hs_r[mask]) and np.array_equal(he[mask], he_r[mask])
        seen_partial |= 0 < den_r < len(inl)
    assert seen_partial


@pytest.mark.parametrize("cap", ["float", "int"])
def test_het42_prune12_variant_bit_exact_against_reference(cap):
    """het42 after the reference's prune_links(c, 12)
    (1,806 -> 588 links): seeded covering chains and uniform mixes scored in
    PARITY are the reference's doubles bit for bit; SCORE within 1e-6 (exact on
    integer capacities)."""
    from _support import RefCluster, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = clusters.CONFIGS["het42-70b-prune12"](cap)
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    assert c.num_links == 588
    rc = RefCluster(d)
    # link walks (the pruned mesh is sparse: plain chains rarely connect) and
    # a uniform-interval mix
    rows = np.concatenate([rc.generate(31, 0, 3000, 0, True, 8),
                           h.generate_host(list(e.kmax), c.num_layers, 32, 0, 1000, 150_000)])
    assert np.array_equal(e.generate_walk_host(31, 0, 3000), rows[:3000])
    vr, sr = rc.score(rows, True, 8)
    v, s = e.score(rows)
    assert np.array_equal(s, sr) and np.array_equal(bits(v), bits(vr))
    assert (vr > 0).mean() > 0.2
    e.mode = "score"
    v2, s2 = e.score(rows)
    assert np.array_equal(s2, sr)
    if cap == "int":
        assert np.array_equal(bits(v2), bits(vr))
    else:
        assert np.all(np.abs(v2 - vr) <= 1e-6 * np.maximum(1.0, np.abs(vr)))


def _huge_dense_cluster():
    """200 nodes, full mesh (40,200 links), 8 layers of 1 GB: the structural
    maximum (32,766 arcs) is far beyond one SM's shared memory."""
    d = clusters.mesh_cluster(200)
    d["model"]["num_layers"] = 8
    d["model"]["param_gb"] = 8.0
    return d


def _two_stage_rows(N, rng, count):
    rows = np.zeros((count, N, 2), np.int16)
    for b in range(count):
        for k in range(N):
            if rng.random() < 0.04 * b:  # later rows leave more nodes idle (smaller graphs)
                continue
            rows[b, k] = (0, 4) if k < N // 2 else (4, 8)
    return rows


def test_graphs_beyond_shared_memory_are_solved_in_the_global_tier():
    """Dense two-stage placements on a 200-node full mesh carry ~10k edges
    (~21k arcs), more than the big shared-memory slot holds: they finish in the
    global-memory tier instead of HELIO_CAND_TOO_LARGE, bit-exact in PARITY
    (values and per-edge flows), within 1e-6 in SCORE."""
    d = _huge_dense_cluster()
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    rows = _two_stage_rows(e.num_nodes, np.random.default_rng(3), 12)
    o = Oracle(d)
    vo, so = o.score(rows)
    assert np.all(so == 0)
    v, s = e.score(rows)
    assert np.array_equal(s, so) and np.array_equal(bits(v), bits(vo))
    e.mode = "score"
    v2, s2 = e.score(rows)
    assert np.array_equal(s2, so)
    assert np.all(np.abs(v2 - vo) <= 1e-6 * np.maximum(1.0, np.abs(vo)))
    e.mode = "parity"
    st, nv, E, val = o.graph(rows[0])
    assert len(E["u"]) > 10_000
    vals, sts, nvs, nes, ints, dbl = e.flows(rows[:1], True, len(E["u"]))
    assert sts[0] == 0 and nes[0] == len(E["u"])
    assert np.array_equal(bits(dbl[0, : nes[0], 1]), bits(E["flow"]))


def test_raw_graph_beyond_shared_memory():
    """A raw graph of 15,000 edges (30,000 arcs, ~360 KB of solver state) runs
    in global memory, bit-exact against the reference's max_flow."""
    from _support import max_flow_raw_oracle
    rng = np.random.default_rng(8)
    n, m = 1500, 15_000
    u = rng.integers(0, n, m).astype(np.int32)
    v = rng.integers(0, n, m).astype(np.int32)
    cap = rng.integers(1, 50, m).astype(np.float64)
    want, wflow = max_flow_raw_oracle(n, 0, n - 1, u, v, cap)
    vals, flows = h.max_flow_raw(np.array([n], np.int32), np.array([0], np.int32), np.array([n - 1], np.int32),
                                 np.array([0, m], np.int64), u, v, cap)
    assert bits(vals)[0] == bits(np.array([want]))[0] and want > 0
    assert np.array_equal(bits(flows), bits(wflow))


def test_generate_trace_matches_reference_fixture():
    z = golden("route_geo24.npz")
    _, inl, outl = h.generate_trace_arrays(len(z["in_len"]), 0.0, "offline", 7)
    assert np.array_equal(inl, z["in_len"]) and np.array_equal(outl, z["out_len"])


def test_iwrr_weights_and_picker_bit_exact():
    z = golden("iwrr.npz")
    off = z["flows_off"]
    for i in range(len(off) - 1):
        a, b = off[i], off[i + 1]
        assert list(h.iwrr_weights(list(z["flows"][a:b]))) == list(z["weights"][a:b])
    po, mo = z["pick_off"], z["pick_moff"]
    for i in range(len(po) - 1):
        w = [int(x) for x in z["pick_w"][po[i]:po[i + 1]]]
        masks = z["pick_masks"][mo[i]:mo[i + 1]]
        want = z["pick_out"][mo[i]:mo[i + 1]]
        p = h.IwrrPicker(w)
        got = [p.next(lambda j, m=int(m): bool((m >> j) & 1)) for m in masks]
        assert got == list(want), i


# --- SCORE mode (value-only Edmonds-Karp) -------------------------------------
# north_star: bit-exact values on integer capacities, within 1e-6 relative on
# float capacities.  Statuses are identical in both modes.
SCORE_REL_TOL = 1e-6


@pytest.mark.parametrize("key", CAND_FIXTURES)
def test_score_mode_against_reference(key):
    z = golden(f"cand_{key}.npz")
    c, e = engine(key)
    e.mode = "score"
    try:
        for partial, vk, sk in ((True, "values_partial", "status_partial"),
                                (False, "values_strict", "status_strict")):
            v, s = e.score(z["rows"], partial)
            assert np.array_equal(s, z[sk]), key
            if key.endswith("_int"):
                assert np.array_equal(bits(v), bits(z[vk])), key
            else:
                ref = z[vk]
                assert np.all(np.abs(v - ref) <= SCORE_REL_TOL * np.maximum(1.0, np.abs(ref))), key
    finally:
        e.mode = "parity"


@pytest.mark.parametrize("name", ["het42-70b", "single24-30b", "geo24", "single24-70b"])
@pytest.mark.parametrize("cap", ["float", "int"])
def test_score_mode_seeded_batches(name, cap):
    d = clusters.CONFIGS[name](cap)
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    e.mode = "score"
    o = Oracle(d)
    rows = np.concatenate([h.generate_host(list(e.kmax), c.num_layers, 31, 0, 3000, 0),
                           h.generate_host(list(e.kmax), c.num_layers, 31, 10**6, 1000, 150000)])
    v, s = e.score(rows)
    vo, so = o.score(rows)
    assert np.array_equal(s, so)
    if cap == "int":
        assert np.array_equal(bits(v), bits(vo))
    else:
        assert np.all(np.abs(v - vo) <= SCORE_REL_TOL * np.maximum(1.0, np.abs(vo)))


def test_score_mode_full_size_matches_parity_mode():
    import torch
    d = clusters.CONFIGS["het42-70b"]("int")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    B = 1_000_000
    pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda")
    e.generate_device(77, 0, B, 50000, pl.data_ptr(), 0)
    vp = torch.empty(B, dtype=torch.float64, device="cuda")
    vs = torch.empty(B, dtype=torch.float64, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    e.score_device(pl.data_ptr(), B, vp.data_ptr(), st.data_ptr(), True, 0)
    e.mode = "score"
    e.score_device(pl.data_ptr(), B, vs.data_ptr(), st.data_ptr(), True, 0)
    torch.cuda.synchronize()
    # integer capacities: the two algorithms agree bit for bit at full size
    assert torch.equal(vp.view(torch.int64), vs.view(torch.int64))


# --- exhaustive placement search (enumerate.hpp:14-77; AC2) ------------------

def test_exhaustive_search_matches_reference():
    z = golden("search_exhaustive.npz")
    for i, key in enumerate(z["keys"]):
        d = golden_cluster(str(key))
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c)
        best, row, scored, total = e.best_exhaustive(bool(z["partial"][i]))
        N = len(d["nodes"])
        assert scored == z["scored"][i], key
        assert bits([best])[0] == bits(z["values"][i : i + 1])[0], key
        assert np.array_equal(row, z["rows"][i][:N]), key
        assert total >= scored


def test_score_best_host_matches_first_max():
    import torch
    c, e = engine("het42-70b_float")
    rows = h.generate_host(list(e.kmax), c.num_layers, 99, 0, 700_000, 80000)
    rows[::97, 0] = (0, 99)  # invalid rows (status 2) must be skipped
    pin = torch.from_numpy(rows).pin_memory()
    for mode in ("parity", "score"):
        e.mode = mode
        try:
            v = torch.empty(len(rows), dtype=torch.float64).pin_memory()
            s = torch.empty(len(rows), dtype=torch.int32).pin_memory()
            best, idx = e.score_best_host_ptr(pin.data_ptr(), len(rows), v.data_ptr(), s.data_ptr(), True)
            vv, ss = v.numpy(), s.numpy()
            ok = (ss == 0) & (vv > 0)
            want = int(np.argmax(np.where(ok, vv, -1.0)))
            assert idx == want and best == vv[want]
            # pageable buffers take the staged path and agree
            v2, s2 = e.score(rows)
            assert np.array_equal(bits(v2), bits(vv)) and np.array_equal(s2, ss)
        finally:
            e.mode = "parity"


def test_walk_generator_device_matches_host_and_syn256_walk_parity():
    import torch
    d = clusters.CONFIGS["syn256-120l"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    B = 2000
    out = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda")
    e.generate_walk_device(7, 100, B, out.data_ptr(), 0)
    torch.cuda.synchronize()
    rows = e.generate_walk_host(7, 100, B)
    assert np.array_equal(out.cpu().numpy(), rows)
    from _support import RefCluster, ref_available
    if ref_available():  # bench.py's reference arm draws the same walks over the reference's ClusterSpec
        assert np.array_equal(RefCluster(d).generate(7, 100, B, 0, True, 4), rows)
    o = Oracle(d)
    sub = rows[:150]
    vo, so = o.score(sub)
    assert (vo > 0).mean() > 0.5  # walks connect on the sparse topology
    v, s = e.score(sub)
    assert np.array_equal(s, so) and np.array_equal(bits(v), bits(vo))
    e.mode = "score"
    v, s = e.score(sub)
    assert np.array_equal(s, so)
    assert np.all(np.abs(v - vo) <= 1e-6 * np.maximum(1.0, np.abs(vo)))


@pytest.mark.parametrize("key", ["het42-70b_float", "geo24_float", "single24-30b_int", "syn256-120l_float"])
def test_split_pipeline_bit_exact_with_fused(key):
    import torch
    c, e = engine(key)
    z = golden(f"cand_{key}.npz")
    rows = np.concatenate([z["rows"], h.generate_host(list(e.kmax), c.num_layers, 3, 0, 3000, 100000)])
    B = len(rows)
    pl = torch.from_numpy(rows).cuda()
    slabs = torch.empty(B * e.csr_slab_bytes, dtype=torch.uint8, device="cuda")
    st1 = torch.empty(B, dtype=torch.int32, device="cuda")
    st2 = torch.empty(B, dtype=torch.int32, device="cuda")
    v = torch.empty(B, dtype=torch.float64, device="cuda")
    e.build_csr_device(pl.data_ptr(), B, slabs.data_ptr(), st1.data_ptr(), True, 0)
    e.solve_csr_device(slabs.data_ptr(), B, v.data_ptr(), st2.data_ptr(), 0)
    torch.cuda.synchronize()
    vf, sf = e.score(rows, True)  # fused PARITY
    s2 = st2.cpu().numpy()
    ok = s2 != 4  # graphs beyond the slab report TOO_LARGE in the split path
    assert np.array_equal(s2[ok], sf[ok]) and np.array_equal(st1.cpu().numpy(), s2)
    assert np.array_equal(bits(v.cpu().numpy()[ok]), bits(vf[ok]))
    if not key.startswith("syn256"):
        # only graphs denser than the small slot (8N arcs) are refused by the split path
        assert ok.mean() > 0.95
    # slab layout: meta V, E, status
    meta = slabs.view(B, -1)[:, :16].cpu().numpy().view(np.int32)
    assert np.array_equal(meta[:, 2], s2)


def test_concurrent_callers_on_one_engine():
    # graphs may be solved concurrently — a shared context
    # serialises its callers, results equal the sequential ones
    from concurrent.futures import ThreadPoolExecutor
    c, e = engine("geo24_float")
    batches = [h.generate_host(list(e.kmax), c.num_layers, 1000 + i, 0, 20_000, 50_000) for i in range(8)]
    want = [e.score(b) for b in batches]

    def job(i):
        return e.score(batches[i]), h.plan_for_placement(c, {"a0": (0, 12), "a1": (12, 24)}).objective

    with ThreadPoolExecutor(8) as ex:
        got = list(ex.map(job, range(8)))
    for (v, s), ((gv, gs), obj) in zip(want, got):
        assert np.array_equal(bits(v), bits(gv)) and np.array_equal(s, gs)
    assert len({obj for _, obj in got}) == 1


def test_device_scoring_on_two_streams_shares_no_scratch():
    # score_device calls on different caller streams must not
    # overlap on the context's shared scratch (work counters, overflow lists)
    import torch
    c, e = engine("het42-70b_float")
    B = 200_000
    pl = [torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda") for _ in range(2)]
    for i in range(2):
        e.generate_device(77 + i, 0, B, 0, pl[i].data_ptr(), 0)
    torch.cuda.synchronize()
    want = []
    for i in range(2):
        v = torch.empty(B, dtype=torch.float64, device="cuda")
        s = torch.empty(B, dtype=torch.int32, device="cuda")
        e.score_device(pl[i].data_ptr(), B, v.data_ptr(), s.data_ptr(), True, 0)
        torch.cuda.synchronize()
        want.append((v.clone(), s.clone()))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for rep in range(3):
        outs = []
        for i in range(2):
            v = torch.full((B,), -1.0, dtype=torch.float64, device="cuda")
            s = torch.full((B,), -1, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            e.score_device(pl[i].data_ptr(), B, v.data_ptr(), s.data_ptr(), True, streams[i].cuda_stream)
            outs.append((v, s))
        torch.cuda.synchronize()
        for (v, s), (wv, ws) in zip(outs, want):
            assert torch.equal(v.view(torch.int64), wv.view(torch.int64)) and torch.equal(s, ws)


# --- solver-boundary sweep: V = 2N + 2 crosses the bitset solver's word counts
# (32 / 64 / 96 / 128 vertices), the N <= 64 cover-mask builders and the
# general per-node-list builder --------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("n,peers", [(15, 0), (16, 0), (31, 0), (32, 0), (47, 0), (48, 0), (63, 0),
                                     (64, 0), (65, 0), (100, 0), (100, 8), (400, 6)])
def test_size_sweep_both_modes_match_oracle(n, peers):
    model = "llama-30b" if n < 40 else "llama2-70b"  # small clusters must still cover the model
    for cap in ("float", "int"):
        d = clusters.mesh_cluster(n, model=model, capacity=cap, peers=peers)
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c)
        if peers:  # sparse: placements that walk existing links
            rows = e.generate_walk_host(78 + n, 0, 800)
        else:
            rows = np.concatenate([h.generate_host(list(e.kmax), c.num_layers, 77 + n, 0, 600, 0),
                                   h.generate_host(list(e.kmax), c.num_layers, 78 + n, 0, 200, 200000)])
        want_v, want_s = Oracle(d).score(rows, True)
        v, s = e.score(rows, True)
        assert np.array_equal(s, want_s)
        assert np.array_equal(bits(v), bits(want_v)), f"PARITY n={n} {cap}"
        e.mode = "score"
        vs_, ss_ = e.score(rows, True)
        assert np.array_equal(ss_, want_s)
        if cap == "int":
            assert np.array_equal(bits(vs_), bits(want_v)), f"SCORE n={n} int"
        else:
            assert np.all(np.abs(vs_ - want_v) <= 1e-6 * np.maximum(1.0, np.abs(want_v))), f"SCORE n={n}"
        assert (want_v > 0).mean() > 0.5, "sweep must exercise non-trivial flows"


def test_push_relabel_solver_on_deep_sparse_graphs():
    """SCORE on graphs over 128 vertices runs the push-relabel solver
    (solve_score.cuh solve_pr): on syn256 link walks it must be bit-exact
    against the reference on integer capacities, within 1e-6 on float ones,
    deterministic run to run, and agree with the Edmonds-Karp solver it
    replaced (HELIO_LARGE_SOLVER=1)."""
    import os
    for cap in ("int", "float"):
        d = clusters.CONFIGS["syn256-120l"](cap)
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c)
        rows = e.generate_walk_host(4242, 0, 3000)
        vo, so = Oracle(d).score(rows[:600])
        e.mode = "score"
        v1, s1 = e.score(rows)
        v2, s2 = e.score(rows)
        assert np.array_equal(bits(v1), bits(v2)) and np.array_equal(s1, s2), "not deterministic"
        assert np.array_equal(s1[:600], so)
        if cap == "int":
            assert np.array_equal(bits(v1[:600]), bits(vo))
        else:
            assert np.all(np.abs(v1[:600] - vo) <= SCORE_REL_TOL * np.maximum(1.0, np.abs(vo)))
        os.environ["HELIO_LARGE_SOLVER"] = "1"
        try:
            e_ek = h.Engine(h.Cluster.from_json(json.dumps(d)))
        finally:
            del os.environ["HELIO_LARGE_SOLVER"]
        e_ek.mode = "score"
        vk, sk = e_ek.score(rows)
        assert np.array_equal(sk, s1)
        if cap == "int":
            assert np.array_equal(bits(vk), bits(v1))
        else:
            assert np.all(np.abs(vk - v1) <= SCORE_REL_TOL * np.maximum(1.0, np.abs(v1)))


def test_dense_placements_take_the_middle_and_big_slots():
    """Placements with replicated stages (the heuristics' petals layout has
    ~5N edges on het42) overflow the small slot (4N edges) into the middle
    tier (8N); fully replicated stages go on to the big slot.  Both tiers must
    match the oracle like the small one."""
    from _support import RefCluster, ref_available, ref_heuristic
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    o = Oracle(d)
    N, L = len(d["nodes"]), c.num_layers
    kmax = list(e.kmax)
    petals, _ = ref_heuristic(RefCluster(d), "petals")
    rng = np.random.default_rng(5)
    rows = [petals]
    for _ in range(600):  # 1-2 node re-assignments of the petals row
        r = petals.copy()
        for _ in range(int(rng.integers(1, 3))):
            k = int(rng.integers(N))
            ln = 1 + int(rng.integers(kmax[k]))
            s = int(rng.integers(0, L - ln + 1))
            r[k] = (s, s + ln)
        rows.append(r)
    for groups in (3, 4, 6):  # every node of a stage on the same 4-layer interval
        r = np.zeros((N, 2), np.int16)
        for k in range(N):
            g = k % groups
            r[k] = (4 * g, 4 * g + 4)
        rows.append(r)
    rows = np.stack(rows).astype(np.int16)
    edges = []
    for r in rows:
        st, nv, E, val = o.graph(r, True)
        edges.append(len(E["u"]) if st == 0 else 0)
    edges = np.array(edges)
    assert (edges > 4 * N).sum() > 100 and (edges > 8 * N).sum() >= 2, "must exercise both tiers"
    want_v, want_s = o.score(rows, True)
    v, s = e.score(rows, True)
    assert np.array_equal(s, want_s) and np.array_equal(bits(v), bits(want_v))
    e.mode = "score"
    vs_, ss_ = e.score(rows, True)
    e.mode = "parity"
    assert np.array_equal(ss_, want_s)
    assert np.all(np.abs(vs_ - want_v) <= SCORE_REL_TOL * np.maximum(1.0, np.abs(want_v)))


@pytest.mark.parametrize("cap", ["float", "int"])
def test_tiny_sparse_cluster_with_many_layers(cap):
    """8 nodes, 3 peers each, 60 layers: fewer structural arcs (2(N + links))
    than the 2L + 2 the N <= 64 builders' cover/start masks need in cap[] —
    every slot is sized for the masks (found by tools/fuzz_parity.py)."""
    d = clusters.mesh_cluster(8, model="llama-30b", capacity=cap, peers=3, seed=5)
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    rows = np.concatenate([e.generate_walk_host(11, 0, 500),
                           h.generate_host(list(e.kmax), c.num_layers, 12, 0, 500, 300000)])
    o = Oracle(d)
    for partial in (True, False):
        want_v, want_s = o.score(rows, partial)
        v, s = e.score(rows, partial)
        assert np.array_equal(s, want_s) and np.array_equal(bits(v), bits(want_v))
        e.mode = "score"
        vs_, ss_ = e.score(rows, partial)
        e.mode = "parity"
        assert np.array_equal(ss_, want_s)
        if cap == "int":
            assert np.array_equal(bits(vs_), bits(want_v))
        else:
            assert np.all(np.abs(vs_ - want_v) <= SCORE_REL_TOL * np.maximum(1.0, np.abs(want_v)))
