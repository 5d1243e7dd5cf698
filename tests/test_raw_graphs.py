"""max_flow on raw graphs (flow_graph.cpp:138-229 accepts any source/sink,
self-loops, parallel edges and zero capacities — AC1).  Seeded random graphs
with float and integer capacities: the C oracle against the compiled
reference (CPU), then the CUDA path against the oracle (GPU), bit for bit."""

import numpy as np
import pytest

from _support import bits, max_flow_raw_oracle, ref, ref_available


def random_graphs(seed, count, max_n, float_caps, allow_same_st=True):
    rng = np.random.default_rng(seed)
    n = rng.integers(1, max_n + 1, count).astype(np.int32)
    s = np.array([rng.integers(x) for x in n], np.int32)
    t = np.array([rng.integers(x) if (allow_same_st and rng.random() < 0.1) or x == 1
                  else (lambda a: a if a != si else (a + 1) % x)(rng.integers(x))
                  for x, si in zip(n, s)], np.int32)
    m = np.array([rng.integers(0, 4 * x + 1) for x in n], np.int64)
    off = np.zeros(count + 1, np.int64)
    off[1:] = np.cumsum(m)
    E = int(off[-1])
    u = np.concatenate([rng.integers(0, x, k) for x, k in zip(n, m)]).astype(np.int32) if E else np.zeros(0, np.int32)
    v = np.concatenate([rng.integers(0, x, k) for x, k in zip(n, m)]).astype(np.int32) if E else np.zeros(0, np.int32)
    if float_caps:
        cap = rng.choice([0.0, 1e-13, 0.1, 1.0 / 3.0, 2.5, 1e3 * rng.random(), 7.0], E) * rng.random(E) * 10
    else:
        cap = rng.integers(0, 60, E).astype(np.float64)
    return dict(n=n, s=s, t=t, off=off, u=u, v=v, cap=np.ascontiguousarray(cap, np.float64))


CASES = [(11, 300, 12, True), (12, 300, 12, False), (13, 60, 90, True), (14, 20, 400, True)]


@pytest.mark.skipif(not ref_available(), reason="compiled reference not built")
@pytest.mark.parametrize("seed,count,max_n,fl", CASES)
def test_oracle_matches_reference_on_random_raw_graphs(seed, count, max_n, fl):
    g = random_graphs(seed, count, max_n, fl)
    lib = ref()
    for i in range(count):
        a, b = g["off"][i], g["off"][i + 1]
        vo, fo = max_flow_raw_oracle(int(g["n"][i]), int(g["s"][i]), int(g["t"][i]),
                                     g["u"][a:b], g["v"][a:b], g["cap"][a:b])
        fr = np.zeros(max(b - a, 1))
        vr = lib.refh_maxflow_raw(int(g["n"][i]), int(g["s"][i]), int(g["t"][i]), int(b - a),
                                  np.ascontiguousarray(g["u"][a:b]) if b > a else np.zeros(1, np.int32),
                                  np.ascontiguousarray(g["v"][a:b]) if b > a else np.zeros(1, np.int32),
                                  np.ascontiguousarray(g["cap"][a:b]) if b > a else np.zeros(1), fr)
        assert bits([vo])[0] == bits([vr])[0], i
        assert np.array_equal(bits(fo), bits(fr[: b - a])), i


@pytest.mark.gpu
@pytest.mark.parametrize("seed,count,max_n,fl", CASES)
def test_gpu_matches_oracle_on_random_raw_graphs(seed, count, max_n, fl):
    import paper_2406_01566_b200 as h
    g = random_graphs(seed, count, max_n, fl)
    vals, flows = h.max_flow_raw(g["n"], g["s"], g["t"], g["off"], g["u"], g["v"], g["cap"])
    for i in range(count):
        a, b = g["off"][i], g["off"][i + 1]
        vo, fo = max_flow_raw_oracle(int(g["n"][i]), int(g["s"][i]), int(g["t"][i]),
                                     g["u"][a:b], g["v"][a:b], g["cap"][a:b])
        assert bits([vo])[0] == bits(vals[i : i + 1])[0], i
        assert np.array_equal(bits(fo), bits(flows[a:b])), i


@pytest.mark.gpu
def test_empty_and_degenerate_batches():
    import json
    import paper_2406_01566_b200 as h
    from paper_2406_01566_b200 import clusters
    c = h.Cluster.from_json(json.dumps(clusters.chain_cluster(2, 2, 1000.0)))
    e = h.Engine(c)
    for mode in ("parity", "score"):
        e.mode = mode
        v, s = e.score(np.zeros((0, 2, 2), np.int16))
        assert len(v) == 0 and len(s) == 0
        v, s = e.score(np.zeros((5, 2, 2), np.int16))  # all idle
        assert np.all(v == 0) and np.all(s == 0)
    vals, flows = h.max_flow_raw(np.array([1], np.int32), np.array([0], np.int32), np.array([0], np.int32),
                                 np.array([0, 0], np.int64), np.zeros(0, np.int32), np.zeros(0, np.int32),
                                 np.zeros(0))
    assert vals[0] == 0.0
