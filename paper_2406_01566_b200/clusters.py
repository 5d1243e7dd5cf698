"""Cluster specifications for the benchmark configurations and the tests.

Every builder returns a dict in the reference's cluster JSON schema
(proj/src/cluster.cpp:102-181: ``model`` / ``coordinator`` / ``nodes`` /
``links`` with ``vram_gb``, ``peak_layer_tokens_per_s``, ``bandwidth_mbps``,
``latency_ms`` ...), so the same text feeds the reference (through its own
``parse_cluster``) and this framework.

Topologies follow the reference's acceptance builders
(proj/tests/acceptance/acceptance_main.cpp:64-228) and SURVEY.md §8(d):

* ``single24``  — dense24's full mesh (acceptance_main.cpp:189-201) with
  4 A100-40, 8 L4-24, 12 T4-16 (configs[0], configs[1]).
* ``het42``     — 42 nodes of 7 GPU types, full mesh at
  10 Gb/s, 1,806 links (configs[2], the headline).
* ``geo24``     — acceptance ``geo24()`` exactly (acceptance_main.cpp:151-184)
  and a 70B variant (configs[3]).
* ``syn256``    — 256 nodes cycling het42's type mix, 120 layers, degree-12
  random peer graph (configs[4]).

``capacity="int"`` selects the integer-capacity variant of SURVEY.md §8(d):
activation_bytes = 15625 (so 8*act = 125000 divides every bandwidth used),
token_bytes = 4, and explicit throughput tables T_j = floor(K / j).
"""

from __future__ import annotations

import json
from typing import Dict, List

# peak layer-tokens/s per device class (acceptance_main.cpp:153-155 for
# A100/L4/T4; the rest per SURVEY.md §8(d)) and VRAM in GB.
GPU_TYPES = {
    "A100": (40.0, 4000.0),
    "V100": (16.0, 1200.0),
    "L4": (24.0, 1000.0),
    "T4": (16.0, 400.0),
    "L4x2": (48.0, 2000.0),
    "T4x2": (32.0, 800.0),
    "T4x4": (64.0, 1600.0),
}

MODELS = {
    "llama2-70b": {"name": "llama2-70b", "num_layers": 80, "param_gb": 140.0,
                   "token_bytes": 4.0, "activation_bytes": 16384.0},
    "llama-30b": {"name": "llama-30b", "num_layers": 60, "param_gb": 65.0,
                  "token_bytes": 4.0, "activation_bytes": 13312.0},
}


def _model(model: str, capacity: str) -> dict:
    m = dict(MODELS[model])
    if capacity == "int":
        m["activation_bytes"] = 15625.0
        m["token_bytes"] = 4.0
    return m


def _max_layers(vram_gb: float, kv_reserve: float, model: dict) -> int:
    """ClusterSpec::max_layers (cluster.cpp:62-68) for a peak-only node."""
    import math
    bpl = model["param_gb"] * 1e9 / int(model["num_layers"])
    k = int(math.floor(vram_gb * 1e9 * (1.0 - kv_reserve) / bpl))
    return min(k, int(model["num_layers"]))


def _node(nid: str, gtype: str, model: dict, capacity: str, vram_gb=None, peak=None) -> dict:
    v, k = GPU_TYPES[gtype]
    vram_gb = v if vram_gb is None else vram_gb
    peak = k if peak is None else peak
    n = {"id": nid, "type": gtype, "vram_gb": vram_gb, "kv_reserve": 0.5}
    if capacity == "int":
        kmax = max(1, _max_layers(vram_gb, 0.5, model))
        n["throughput_table"] = {str(j): float(int(peak) // j) for j in range(1, kmax + 1)}
    else:
        n["peak_layer_tokens_per_s"] = peak
    return n


def _biline(links: List[dict], a: str, b: str, bw_bps: float, lat_s: float) -> None:
    """acceptance_main.cpp:77-80: one link each way."""
    links.append({"src": a, "dst": b, "bandwidth_mbps": bw_bps / 1e6, "latency_ms": lat_s * 1e3})
    links.append({"src": b, "dst": a, "bandwidth_mbps": bw_bps / 1e6, "latency_ms": lat_s * 1e3})


def single24(model: str = "llama2-70b", capacity: str = "float") -> dict:
    """dense24's topology (acceptance_main.cpp:189-201) with 40 GB A100s."""
    m = _model(model, capacity)
    nodes = []
    for i in range(4):
        nodes.append(_node(f"a{i}", "A100", m, capacity))
    for i in range(8):
        nodes.append(_node(f"l{i}", "L4", m, capacity))
    for i in range(12):
        nodes.append(_node(f"t{i}", "T4", m, capacity))
    links: List[dict] = []
    for n in nodes:
        _biline(links, "coord", n["id"], 10e9, 0.0002)
    for i in range(len(nodes)):
        for j in range(i + 1, len(nodes)):
            chain = nodes[i]["type"] == nodes[j]["type"] and j == i + 1
            _biline(links, nodes[i]["id"], nodes[j]["id"], 10e9, 0.0002 if chain else 0.001)
    return {"model": m, "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


HET42_MIX = [("A100", 4), ("V100", 6), ("L4", 8), ("T4", 10), ("L4x2", 4), ("T4x2", 6), ("T4x4", 4)]


def het42(model: str = "llama2-70b", capacity: str = "float") -> dict:
    """42-node, 7-type cluster, full mesh at 10 Gb/s: 1,806 links."""
    m = _model(model, capacity)
    nodes = []
    for gtype, count in HET42_MIX:
        for i in range(count):
            nodes.append(_node(f"{gtype.lower()}-{i}", gtype, m, capacity))
    links: List[dict] = []
    for n in nodes:
        _biline(links, "coord", n["id"], 10e9, 0.0002)
    for i in range(len(nodes)):
        for j in range(i + 1, len(nodes)):
            _biline(links, nodes[i]["id"], nodes[j]["id"], 10e9, 0.001)
    return {"model": m, "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def geo24(variant: str = "m24", capacity: str = "float") -> dict:
    """acceptance_main.cpp:151-184 exactly (variant "m24"); variant "70b" swaps
    in LLaMA-2-70B with 40 GB A100s / 24 GB L4s / 16 GB T4s and 100 Mb/s,
    50 ms inter-region links."""
    if variant == "m24":
        m = {"name": "m24", "num_layers": 24, "param_gb": 24.0, "token_bytes": 4.0,
             "activation_bytes": 16384.0}
        if capacity == "int":
            m["activation_bytes"] = 15625.0
        vr = {"A100": 24.0, "L4": 12.0, "T4": 6.0}
        wan_bw, wan_lat = 12e6, 0.05
    else:
        m = _model("llama2-70b", capacity)
        vr = {"A100": 40.0, "L4": 24.0, "T4": 16.0}
        wan_bw, wan_lat = 100e6, 0.05
    pk = {"A100": 4000.0, "L4": 1000.0, "T4": 400.0}

    def mk(nid: str, t: str) -> dict:
        return _node(nid, t, m, capacity, vram_gb=vr[t], peak=pk[t])

    order = [("a0", "A100"), ("bl0", "L4"), ("cl0", "L4"), ("bt0", "T4"), ("ct0", "T4"),
             ("a1", "A100"), ("bt1", "T4"), ("cl1", "L4"), ("bt2", "T4"), ("ct1", "T4"),
             ("a2", "A100"), ("bl1", "L4"), ("cl2", "L4"), ("bt3", "T4"), ("ct2", "T4"),
             ("a3", "A100"), ("bt4", "T4"), ("cl3", "L4"), ("bt5", "T4"), ("ct3", "T4"),
             ("cl4", "L4"), ("bt6", "T4"), ("cl5", "L4"), ("bt7", "T4")]
    nodes = [mk(i, t) for i, t in order]
    ra = [n["id"] for n in nodes if n["id"][0] == "a"]
    rb = [n["id"] for n in nodes if n["id"][0] == "b"]
    rc = [n["id"] for n in nodes if n["id"][0] == "c"]
    links: List[dict] = []
    for n in nodes:
        fast = n["id"][0] == "a"
        _biline(links, "coord", n["id"], 10e9 if fast else 100e6, 0.0002 if fast else 0.02)

    def ring(r: List[str]) -> None:
        for i in range(len(r)):
            _biline(links, r[i], r[(i + 1) % len(r)], 10e9, 0.0002)
        _biline(links, r[0], r[len(r) // 2], 10e9, 0.0002)
        if len(r) > 4:
            _biline(links, r[1], r[len(r) // 2 + 1], 10e9, 0.0002)

    ring(ra)
    ring(rb)
    ring(rc)

    def wan(x: List[str], y: List[str]) -> None:
        for u in x:
            for v in y:
                _biline(links, u, v, wan_bw, wan_lat)

    wan(ra, rb)
    wan(ra, rc)
    wan(rb, rc)
    return {"model": m, "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def syn256(capacity: str = "float", seed: int = 256) -> dict:
    """256 nodes cycling het42's type mix, 120 layers, param_gb=210
    (1.75 GB/layer), coordinator <-> every node, and each node linked (both
    ways) to 12 seeded random peers."""
    m = {"name": "syn120", "num_layers": 120, "param_gb": 210.0, "token_bytes": 4.0,
         "activation_bytes": 15625.0 if capacity == "int" else 16384.0}
    mix = [t for t, c in HET42_MIX for _ in range(c)]
    nodes = [_node(f"n{i:03d}", mix[i % len(mix)], m, capacity) for i in range(256)]
    links: List[dict] = []
    for n in nodes:
        _biline(links, "coord", n["id"], 10e9, 0.0002)
    seen = set()
    state = seed
    for i in range(256):
        picked = 0
        while picked < 12:
            state = _splitmix64(state)
            j = state % 256
            if j == i:
                continue
            key = (min(i, j), max(i, j))
            if key in seen:
                picked += 1  # already linked from the other side: counts toward degree
                continue
            seen.add(key)
            _biline(links, nodes[i]["id"], nodes[j]["id"], 10e9, 0.001)
            picked += 1
    return {"model": m, "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def mesh_cluster(n: int, model: str = "llama2-70b", capacity: str = "float", peers: int = 0,
                 seed: int = 1) -> dict:
    """n nodes cycling het42's type mix, coordinator <-> every node, and a full
    mesh (peers == 0) or `peers` seeded random neighbours per node: the
    size sweep behind the solver-boundary tests (V = 2n + 2 crosses 32, 64,
    96 and 128)."""
    m = _model(model, capacity)
    mix = [t for t, c in HET42_MIX for _ in range(c)]
    nodes = [_node(f"m{i:03d}", mix[i % len(mix)], m, capacity) for i in range(n)]
    links: List[dict] = []
    for x in nodes:
        _biline(links, "coord", x["id"], 10e9, 0.0002)
    if peers <= 0:
        for i in range(n):
            for j in range(i + 1, n):
                _biline(links, nodes[i]["id"], nodes[j]["id"], 10e9, 0.001)
    else:
        seen = set()
        state = seed
        for i in range(n):
            for _ in range(peers):
                state = _splitmix64(state)
                j = state % n
                key = (min(i, j), max(i, j))
                if j == i or key in seen:
                    continue
                seen.add(key)
                _biline(links, nodes[i]["id"], nodes[j]["id"], 10e9, 0.001)
    return {"model": m, "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def make_node(nid: str, hold_layers: int, peak: float, gtype: str = "gpu") -> dict:
    """test_support.hpp:11-20: k layers at 1 GB beside the KV half."""
    return {"id": nid, "type": gtype, "vram_gb": 2.0 * hold_layers + 1.0, "kv_reserve": 0.5,
            "peak_layer_tokens_per_s": peak}


def make_link(src: str, dst: str, bw_bps: float, lat_s: float = 0.001) -> dict:
    """test_support.hpp:22-30."""
    return {"src": src, "dst": dst, "bandwidth_mbps": bw_bps / 1e6, "latency_ms": lat_s * 1e3}


def chain_cluster(stages: int, layers_per_stage: int, peak: float, bw_bps: float = 10e9) -> dict:
    """test_support.hpp:33-48: coord -> n0 -> n1 -> ... -> coord."""
    L = stages * layers_per_stage
    nodes = [make_node(f"n{i}", layers_per_stage, peak) for i in range(stages)]
    links = [make_link("coord", "n0", bw_bps)]
    for i in range(stages - 1):
        links.append(make_link(f"n{i}", f"n{i + 1}", bw_bps))
    links.append(make_link(f"n{stages - 1}", "coord", bw_bps))
    return {"model": {"name": "toy", "num_layers": L, "param_gb": float(L)},
            "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def fan3() -> dict:
    """acceptance_main.cpp:138-146: three full-model replicas (AC8)."""
    nodes = [
        {"id": "p0", "type": "A", "vram_gb": 6.0, "kv_reserve": 0.5, "peak_layer_tokens_per_s": 640.0},
        {"id": "p1", "type": "B", "vram_gb": 6.0, "kv_reserve": 0.5, "peak_layer_tokens_per_s": 380.0},
        {"id": "p2", "type": "C", "vram_gb": 6.0, "kv_reserve": 0.5, "peak_layer_tokens_per_s": 260.0},
    ]
    links: List[dict] = []
    for n in nodes:
        _biline(links, "coord", n["id"], 10e9, 0.0002)
    return {"model": {"name": "m2", "num_layers": 2, "param_gb": 2.0, "token_bytes": 4.0,
                      "activation_bytes": 16384.0},
            "coordinator": {"id": "coord"}, "nodes": nodes, "links": links}


def het42_prune12(capacity: str = "float") -> dict:
    """het42 after the reference's prune_links(c, 12) (placement.cpp:230-332;
    SURVEY.md §8(d) item 3): 1,806 -> 588 links, average degree 12.  The JSON
    is the reference's own output (tests/golden/make_workloads.py), shipped
    as data; prune_links(cluster, 12) reproduces it on the engine side."""
    import gzip
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", f"het42-70b-prune12_{capacity}.json.gz")
    with gzip.open(path, "rt") as f:
        return json.load(f)


CONFIGS: Dict[str, callable] = {
    "single24-70b": lambda cap="float": single24("llama2-70b", cap),
    "single24-30b": lambda cap="float": single24("llama-30b", cap),
    "het42-70b": lambda cap="float": het42("llama2-70b", cap),
    "geo24": lambda cap="float": geo24("m24", cap),
    "geo24-70b": lambda cap="float": geo24("70b", cap),
    "syn256-120l": lambda cap="float": syn256(cap),
    "het42-70b-prune12": het42_prune12,
}


def cluster_json(name: str, capacity: str = "float") -> str:
    return json.dumps(CONFIGS[name](capacity))
