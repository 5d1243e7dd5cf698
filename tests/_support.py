"""Test infrastructure: ctypes access to the CPU oracle (oracle/_ref/liboracle.so,
the plain-C restatement) and to the compiled reference (oracle/_ref/libhelio_ref.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""

from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_ref", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhelio_ref.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")

_i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OraCluster(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32), ("num_links", C.c_int32), ("num_layers", C.c_int32),
        ("param_bytes", C.c_double), ("token_bytes", C.c_double), ("activation_bytes", C.c_double),
        ("kv_bytes_per_token_layer", C.c_double),
        ("vram_bytes", C.c_void_p), ("kv_reserve", C.c_void_p), ("peak_layer_tokens", C.c_void_p),
        ("nic_in_bps", C.c_void_p), ("nic_out_bps", C.c_void_p), ("table_off", C.c_void_p),
        ("table_val", C.c_void_p), ("lex_rank", C.c_void_p), ("link_src", C.c_void_p),
        ("link_dst", C.c_void_p), ("link_bw", C.c_void_p),
    ]


class ClusterArrays:
    """Numeric view of a cluster JSON dict, computed with the reference's parse
    arithmetic (cluster.cpp:120-176: *1e9 for GB/Gbps, *1e6 for Mbps)."""

    def __init__(self, d: dict):
        m = d["model"]
        self.dict = d
        self.ids = [n["id"] for n in d["nodes"]]
        self.coord = d["coordinator"]["id"]
        self.N = len(self.ids)
        self.L = int(float(m["num_layers"]))
        self.param_bytes = float(m["param_gb"]) * 1e9
        self.token_bytes = float(m.get("token_bytes", 4.0))
        self.activation_bytes = float(m.get("activation_bytes", 16384.0))
        self.kv = float(m.get("kv_bytes_per_token_layer", 0.0))
        nodes = d["nodes"]
        self.vram = np.array([float(n["vram_gb"]) * 1e9 for n in nodes], np.float64)
        self.kv_reserve = np.array([float(n.get("kv_reserve", 0.5)) for n in nodes], np.float64)
        self.peak = np.array([float(n.get("peak_layer_tokens_per_s", 0.0)) for n in nodes], np.float64)
        self.nic_in = np.array([float(n.get("nic_in_gbps", 0.0)) * 1e9 for n in nodes], np.float64)
        self.nic_out = np.array([float(n.get("nic_out_gbps", 0.0)) * 1e9 for n in nodes], np.float64)
        off = [0]
        vals = []
        for n in nodes:
            t = n.get("throughput_table") or {}
            for j in range(1, len(t) + 1):
                vals.append(float(t[str(j)]))
            off.append(len(vals))
        self.table_off = np.array(off, np.int32)
        self.table_val = np.array(vals if vals else [0.0], np.float64)
        order = sorted(range(self.N), key=lambda i: self.ids[i].encode())
        self.lex_rank = np.zeros(self.N, np.int32)
        for r, i in enumerate(order):
            self.lex_rank[i] = r
        pos = {nid: i for i, nid in enumerate(self.ids)}

        def ep(x):
            return -1 if x == self.coord else pos.get(x, -2)

        links = d["links"]
        self.link_src = np.array([ep(l["src"]) for l in links], np.int32)
        self.link_dst = np.array([ep(l["dst"]) for l in links], np.int32)
        self.link_bw = np.array([float(l["bandwidth_mbps"]) * 1e6 for l in links], np.float64)
        self.M = len(links)

    def ora(self) -> OraCluster:
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        return OraCluster(self.N, self.M, self.L, self.param_bytes, self.token_bytes,
                          self.activation_bytes, self.kv, p(self.vram), p(self.kv_reserve),
                          p(self.peak), p(self.nic_in), p(self.nic_out), p(self.table_off),
                          p(self.table_val), p(self.lex_rank), p(self.link_src), p(self.link_dst),
                          p(self.link_bw))


_oracle = None


def oracle():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        oc = C.POINTER(OraCluster)
        lib.ora_max_layers.argtypes = [oc, C.c_int]
        lib.ora_max_layers.restype = C.c_int
        lib.ora_compute_edge_capacity.argtypes = [oc, C.c_int, C.c_int]
        lib.ora_compute_edge_capacity.restype = C.c_double
        lib.ora_build.argtypes = [oc, _i16p, C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p, _i32p,
                                  _i32p, _i32p, _f64p]
        lib.ora_build.restype = C.c_int
        lib.ora_max_flow.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _f64p, _f64p]
        lib.ora_max_flow.restype = C.c_double
        lib.ora_score.argtypes = [oc, _i16p, C.c_int64, C.c_int, _f64p, _i32p]
        lib.ora_score.restype = C.c_int
        lib.ora_iwrr_weights.argtypes = [_f64p, C.c_int, _i64p]
        lib.ora_plan.argtypes = [oc, _i16p, C.c_int, C.c_int, _i32p, _i32p, _f64p, _i32p, _i32p, _f64p]
        lib.ora_plan.restype = C.c_int
        lib.ora_route.argtypes = [oc, _i16p, C.c_int, C.c_int64, _i32p, _i32p, C.c_int, _i32p, _i32p,
                                  _i32p, _i32p]
        lib.ora_route.restype = C.c_int64
        _oracle = lib
    return _oracle


class Oracle:
    """The C restatement bound to one cluster."""

    def __init__(self, d: dict):
        self.ca = ClusterArrays(d)
        self.oc = self.ca.ora()
        self.lib = oracle()

    @property
    def N(self):
        return self.ca.N

    def kmax(self):
        return [self.lib.ora_max_layers(C.byref(self.oc), k) for k in range(self.ca.N)]

    def score(self, rows: np.ndarray, partial=True):
        rows = np.ascontiguousarray(rows, np.int16)
        B = rows.shape[0]
        v = np.zeros(B, np.float64)
        s = np.zeros(B, np.int32)
        self.lib.ora_score(C.byref(self.oc), rows, B, int(partial), v, s)
        return v, s

    def graph(self, row: np.ndarray, partial=True):
        """-> (status, nv, edges dict of arrays incl. flow, value)."""
        row = np.ascontiguousarray(row, np.int16)
        max_e = self.ca.N + self.ca.M + 1
        a = {k: np.zeros(max_e, np.int32) for k in ("u", "v", "kind", "es", "ee")}
        cap = np.zeros(max_e, np.float64)
        nv = np.zeros(1, np.int32)
        ne = np.zeros(1, np.int32)
        st = self.lib.ora_build(C.byref(self.oc), row, int(partial), max_e, nv, ne, a["u"], a["v"],
                                a["kind"], a["es"], a["ee"], cap)
        if st != 0:
            return st, 0, None, 0.0
        E = int(ne[0])
        edges = {k: x[:E].copy() for k, x in a.items()}
        edges["cap"] = cap[:E].copy()
        flow = np.zeros(E, np.float64)
        val = self.lib.ora_max_flow(int(nv[0]), 0, 1, E, edges["u"], edges["v"], edges["cap"], flow)
        edges["flow"] = flow
        return 0, int(nv[0]), edges, val

    def plan(self, row, partial=True):
        row = np.ascontiguousarray(row, np.int16)
        max_e = self.ca.N + self.ca.M + 1
        src = np.zeros(max_e, np.int32)
        dst = np.zeros(max_e, np.int32)
        es = np.zeros(max_e, np.int32)
        ee = np.zeros(max_e, np.int32)
        fl = np.zeros(max_e, np.float64)
        obj = np.zeros(1, np.float64)
        n = self.lib.ora_plan(C.byref(self.oc), row, int(partial), max_e, src, dst, fl, es, ee, obj)
        if n < 0:
            return n, None, 0.0
        return n, dict(src=src[:n], dst=dst[:n], es=es[:n], ee=ee[:n], flow=fl[:n]), float(obj[0])

    def route(self, row, in_len, out_len, partial=True, max_hops=None):
        row = np.ascontiguousarray(row, np.int16)
        R = len(in_len)
        H = max_hops or self.ca.L
        nh = np.zeros(R, np.int32)
        hn = np.full(R * H, -9, np.int32)
        hs = np.zeros(R * H, np.int32)
        he = np.zeros(R * H, np.int32)
        den = self.lib.ora_route(C.byref(self.oc), row, int(partial), R,
                                 np.ascontiguousarray(in_len, np.int32),
                                 np.ascontiguousarray(out_len, np.int32), H, nh, hn, hs, he)
        return den, nh, hn.reshape(R, H), hs.reshape(R, H), he.reshape(R, H)


def max_flow_raw_oracle(n, s, t, u, v, cap):
    u = np.ascontiguousarray(u, np.int32)
    v = np.ascontiguousarray(v, np.int32)
    cap = np.ascontiguousarray(cap, np.float64)
    flow = np.zeros(max(len(u), 1), np.float64)
    val = oracle().ora_max_flow(n, s, t, len(u), u, v, cap, flow)
    return val, flow[: len(u)]


def iwrr_weights_oracle(flows):
    f = np.ascontiguousarray(flows, np.float64)
    w = np.zeros(len(f), np.int64)
    oracle().ora_iwrr_weights(f, len(f), w)
    return w


# --- compiled reference (oracle/_ref/libhelio_ref.so) -------------------------

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.refh_cluster_from_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        lib.refh_cluster_from_json.restype = C.c_void_p
        lib.refh_cluster_free.argtypes = [C.c_void_p]
        lib.refh_max_layers.argtypes = [C.c_void_p, C.c_int]
        lib.refh_max_layers.restype = C.c_int
        lib.refh_compute_edge_capacity.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.refh_compute_edge_capacity.restype = C.c_double
        lib.refh_graph.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p,
                                   _i32p, _i32p, _i32p, _f64p, _f64p, _f64p, C.c_char_p, C.c_int]
        lib.refh_graph.restype = C.c_int
        lib.refh_score.argtypes = [C.c_void_p, _i16p, C.c_int64, C.c_int, C.c_int, _f64p, _i32p]
        lib.refh_score.restype = C.c_int
        lib.refh_solve_only.argtypes = [C.c_void_p, _i16p, C.c_int64, C.c_int, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.refh_solve_only.restype = C.c_int64
        lib.refh_generate.argtypes = [C.c_void_p, C.c_uint64, C.c_int64, C.c_int64, C.c_uint32, C.c_int,
                                      C.c_int, _i16p]
        lib.refh_generate.restype = C.c_int
        lib.refh_maxflow_raw.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _i32p, _f64p, _f64p]
        lib.refh_maxflow_raw.restype = C.c_double
        lib.refh_ac1_graphs.argtypes = [C.c_uint64, C.c_int, _i32p, _i32p, _i32p, _i32p, _i32p, _f64p,
                                        C.c_int64]
        lib.refh_ac1_graphs.restype = C.c_int64
        lib.refh_testflow_graphs.argtypes = [C.c_uint64, C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p,
                                             _f64p, C.c_int64]
        lib.refh_testflow_graphs.restype = C.c_int64
        lib.refh_iwrr_weights.argtypes = [_f64p, C.c_int, _i64p]
        lib.refh_picker_seq.argtypes = [_i64p, C.c_int, C.c_int, _u64p, _i32p]
        lib.refh_plan.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_int, _i32p, _i32p, _f64p, _i32p,
                                  _i32p, _f64p]
        lib.refh_plan.restype = C.c_int
        lib.refh_route.argtypes = [C.c_void_p, _i16p, C.c_int, C.c_uint64, C.c_int64, _i32p, _i32p,
                                   C.c_int, _i32p, _i32p, _i32p, _i32p]
        lib.refh_route.restype = C.c_int64
        lib.refh_trace.argtypes = [C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_double, C.c_double,
                                   C.c_int, C.c_int, _f64p, _i32p, _i32p]
        lib.refh_trace.restype = C.c_int
        lib.refh_plan_milp.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_long, C.c_double,
                                       C.c_int, _i16p, _i32p, _f64p, _i64p]
        lib.refh_plan_milp.restype = C.c_double
        _ref = lib
    return _ref


class RefCluster:
    """A ClusterSpec parsed by the reference's own parse_cluster."""

    def __init__(self, d: dict):
        err = C.create_string_buffer(512)
        self.lib = ref()
        self.h = self.lib.refh_cluster_from_json(json.dumps(d).encode(), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.N = len(d["nodes"])
        self.M = len(d["links"])
        self.L = int(d["model"]["num_layers"])

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.refh_cluster_free(self.h)

    def score(self, rows, partial=True, threads=1):
        rows = np.ascontiguousarray(rows, np.int16)
        B = rows.shape[0]
        v = np.zeros(B, np.float64)
        s = np.zeros(B, np.int32)
        self.lib.refh_score(self.h, rows, B, int(partial), threads, v, s)
        return v, s

    def generate(self, seed, first, n, ppm=0, walk=False, threads=1):
        """bench.py's workload rows G(seed, i) restated over the reference's
        ClusterSpec (refh_generate; the reference arm's input generator)."""
        out = np.zeros((n, self.N, 2), np.int16)
        self.lib.refh_generate(self.h, seed, first, n, ppm, int(walk), threads, out)
        return out

    def graph(self, row, partial=True):
        row = np.ascontiguousarray(row, np.int16)
        max_e = self.N + self.M + 1
        a = {k: np.zeros(max_e, np.int32) for k in ("u", "v", "kind", "es", "ee")}
        cap = np.zeros(max_e, np.float64)
        flow = np.zeros(max_e, np.float64)
        nv = np.zeros(1, np.int32)
        ne = np.zeros(1, np.int32)
        val = np.zeros(1, np.float64)
        err = C.create_string_buffer(512)
        st = self.lib.refh_graph(self.h, row, int(partial), max_e, nv, ne, a["u"], a["v"], a["kind"],
                                 a["es"], a["ee"], cap, flow, val, err, 512)
        if st != 0:
            return st, 0, None, 0.0, err.value.decode()
        E = int(ne[0])
        edges = {k: x[:E].copy() for k, x in a.items()}
        edges["cap"] = cap[:E].copy()
        edges["flow"] = flow[:E].copy()
        return 0, int(nv[0]), edges, float(val[0]), ""

    def plan(self, row, partial=True):
        row = np.ascontiguousarray(row, np.int16)
        max_e = self.N + self.M + 1
        src = np.zeros(max_e, np.int32)
        dst = np.zeros(max_e, np.int32)
        es = np.zeros(max_e, np.int32)
        ee = np.zeros(max_e, np.int32)
        fl = np.zeros(max_e, np.float64)
        obj = np.zeros(1, np.float64)
        n = self.lib.refh_plan(self.h, row, int(partial), max_e, src, dst, fl, es, ee, obj)
        if n < 0:
            return n, None, 0.0
        return n, dict(src=src[:n], dst=dst[:n], es=es[:n], ee=ee[:n], flow=fl[:n]), float(obj[0])

    def route(self, row, in_len, out_len, partial=True, seed=7, max_hops=None):
        row = np.ascontiguousarray(row, np.int16)
        R = len(in_len)
        H = max_hops or self.L
        nh = np.zeros(R, np.int32)
        hn = np.full(R * H, -9, np.int32)
        hs = np.zeros(R * H, np.int32)
        he = np.zeros(R * H, np.int32)
        den = self.lib.refh_route(self.h, row, int(partial), seed, R,
                                  np.ascontiguousarray(in_len, np.int32),
                                  np.ascontiguousarray(out_len, np.int32), H, nh, hn, hs, he)
        return den, nh, hn.reshape(R, H), hs.reshape(R, H), he.reshape(R, H)


HYB_SO = os.path.join(ROOT, "oracle", "_ref", "libhelio_hybrid.so")


def plan_milp(lib, prefix, handle, N, partial, gap=0.0, lex=False, node_budget=-1, prune=0.0, warm=True):
    """plan_placement through a harness (refh_ = pure reference, hyb_ = the
    reference planner over the B200 drop-in).  -> (objective, row, status,
    best_bound, nodes_explored)."""
    fn = getattr(lib, prefix + "plan_milp")
    row = np.zeros((N, 2), np.int16)
    st = np.zeros(1, np.int32)
    bb = np.zeros(1, np.float64)
    ne = np.zeros(1, np.int64)
    obj = fn(handle, int(partial), gap, int(lex), node_budget, prune, int(warm), row, st, bb, ne)
    return obj, row, int(st[0]), float(bb[0]), int(ne[0])


def hybrid():
    lib = C.CDLL(HYB_SO)
    lib.hyb_cluster_from_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
    lib.hyb_cluster_from_json.restype = C.c_void_p
    lib.hyb_cluster_free.argtypes = [C.c_void_p]
    lib.hyb_plan_milp.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_long, C.c_double,
                                  C.c_int, _i16p, _i32p, _f64p, _i64p]
    lib.hyb_plan_milp.restype = C.c_double
    return lib


def ref_trace(count, seed, mean_in=763.0, mean_out=232.0, max_in=2048, max_out=1024, rate=0.0,
              online=False):
    arr = np.zeros(count, np.float64)
    i = np.zeros(count, np.int32)
    o = np.zeros(count, np.int32)
    ref().refh_trace(count, rate, int(online), seed, mean_in, mean_out, max_in, max_out, arr, i, o)
    return arr, i, o


def ref_raw_graphs(kind: str):
    """AC1 (acceptance_main.cpp:266-295) or test_flow (test_flow.cpp:163-188) graph sets."""
    lib = ref()
    if kind == "ac1":
        count, seed = 1000, 424201
        n = np.zeros(count, np.int32)
        t = np.zeros(count, np.int32)
        m = np.zeros(count, np.int32)
        tot = lib.refh_ac1_graphs(seed, count, n, t, m, np.zeros(1, np.int32), np.zeros(1, np.int32),
                                  np.zeros(1, np.float64), 0)
        eu = np.zeros(tot, np.int32)
        ev = np.zeros(tot, np.int32)
        ec = np.zeros(tot, np.float64)
        lib.refh_ac1_graphs(seed, count, n, t, m, eu, ev, ec, tot)
        s = np.zeros(count, np.int32)
    else:
        count, seed = 400, 20240811
        n = np.zeros(count, np.int32)
        m = np.zeros(count, np.int32)
        tot = lib.refh_testflow_graphs(seed, count, 19, n, m, np.zeros(1, np.int32),
                                       np.zeros(1, np.int32), np.zeros(1, np.float64), 0)
        eu = np.zeros(tot, np.int32)
        ev = np.zeros(tot, np.int32)
        ec = np.zeros(tot, np.float64)
        lib.refh_testflow_graphs(seed, count, 19, n, m, eu, ev, ec, tot)
        s = np.zeros(count, np.int32)
        t = np.ones(count, np.int32)
    off = np.zeros(count + 1, np.int64)
    off[1:] = np.cumsum(m)
    return dict(n=n, s=s, t=t, off=off, u=eu, v=ev, cap=ec)


# --- golden fixtures (tests/golden/, generated from the compiled reference) --

_clusters = None


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def golden_cluster(key: str) -> dict:
    """Cluster dict a fixture was generated with (tests/golden/clusters.json.gz)."""
    global _clusters
    if _clusters is None:
        import gzip
        with gzip.open(os.path.join(GOLDEN, "clusters.json.gz"), "rt") as f:
            _clusters = json.load(f)
    return _clusters[key]


CAND_FIXTURES = [f"{n}_{c}" for n in ("single24-70b", "single24-30b", "het42-70b", "geo24",
                                       "geo24-70b", "syn256-120l") for c in ("float", "int")]


def bits(a):
    """Exact bit pattern of a float64 array (for bit-exact comparisons)."""
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def neighbour_moves(kmax, L, swaps=False):
    """helio_gpu_local_search's neighbourhood in its order: single-node moves,
    node-major, per node the choices of enumerate.hpp:21-28 (idle, then [s, e)
    with e - s <= k_i in (s, e) order); then (swaps) every exchange of two
    nodes' intervals, (i, j) with i < j in order.
    -> (node int[C], start int16[C], end int16[C], partner int[C]): partner
    >= 0 marks a swap of `node` and `partner` (start/end unused)."""
    node, st, en, pa = [], [], [], []
    for i, k in enumerate(kmax):
        node.append(i); st.append(0); en.append(0); pa.append(-1)
        for s in range(L):
            for e in range(s + 1, min(L, s + k) + 1):
                node.append(i); st.append(s); en.append(e); pa.append(-1)
    if swaps:
        for i in range(len(kmax)):
            for j in range(i + 1, len(kmax)):
                node.append(i); st.append(0); en.append(0); pa.append(j)
    return np.array(node), np.array(st, np.int16), np.array(en, np.int16), np.array(pa)


def local_search_oracle(score, kmax, L, seed_row, max_moves=-1, swaps=True):
    """CPU statement of the device local search over any scorer
    score(rows int16[B,N,2]) -> (values, status): best-improvement moves over
    neighbour_moves(), first strict maximum over status-OK positive values
    (enumerate.hpp:59).  -> (value, row, moves, scored)."""
    node, st, en, pa = neighbour_moves(kmax, L, swaps)
    C_ = len(node)
    single = pa < 0
    cur = np.array(seed_row, np.int16).copy()
    v, s = score(cur[None])
    assert s[0] == 0, "seed must validate"
    value, scored, moves = float(v[0]), 1, 0
    idx = np.arange(C_)
    while max_moves < 0 or moves < max_moves:
        rows = np.repeat(cur[None], C_, axis=0)
        rows[idx[single], node[single], 0] = st[single]
        rows[idx[single], node[single], 1] = en[single]
        sw = ~single
        rows[idx[sw], node[sw]] = cur[pa[sw]]
        rows[idx[sw], pa[sw]] = cur[node[sw]]
        vals, sts = score(rows)
        scored += C_
        ok = (sts == 0) & (vals > 0)
        if not ok.any():
            break
        bi = int(np.argmax(np.where(ok, vals, -np.inf)))
        if not vals[bi] > value:
            break
        value = float(vals[bi])
        cur = rows[bi].copy()
        moves += 1
    return value, cur, moves, scored


def ref_heuristic(rc: "RefCluster", method: str):
    """The reference's swarm / petals / sp placement as an int16 [N][2] row plus
    its warnings (or the exception text as a ValueError)."""
    lib = ref()
    lib.refh_heuristic.argtypes = [C.c_void_p, C.c_int, _i16p, C.c_char_p, C.c_int]
    lib.refh_heuristic.restype = C.c_int
    row = np.zeros((rc.N, 2), np.int16)
    buf = C.create_string_buffer(8192)
    n = lib.refh_heuristic(rc.h, {"swarm": 0, "petals": 1, "sp": 2}[method], row, buf, 8192)
    text = buf.value.decode()
    if n < 0:
        raise ValueError(text)
    return row, (text.split("\n") if n > 0 else [])
