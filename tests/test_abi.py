"""CPU: the C-ABI library loads and exports every entry point include/helio_gpu.h
declares; the Python extension imports; without a GPU the engine refuses to run
(no CPU fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "helio_gpu.h")
LIB = os.path.join(ROOT, "paper_2406_01566_b200", "lib", "libhelio_gpu.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(helio_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("helio_gpu_create", "helio_gpu_set_cluster", "helio_gpu_score", "helio_gpu_score_host",
              "helio_gpu_flows_host", "helio_gpu_maxflow_raw_host", "helio_gpu_argmax",
              "helio_gpu_route_host", "helio_gpu_generate", "helio_generate_host"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_extension_imports_and_mirrors_reference_names():
    import paper_2406_01566_b200 as h
    for name in ("Cluster", "Plan", "ParseError", "ValidationError", "max_flow_value",
                 "plan_for_placement"):
        assert hasattr(h, name)
    assert issubclass(h.ValidationError, ValueError)
    assert issubclass(h.ParseError, ValueError)


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="only meaningful without a GPU")
def test_no_cpu_fallback_without_gpu():
    import paper_2406_01566_b200 as h
    from paper_2406_01566_b200 import clusters
    c = h.Cluster.from_json(clusters.cluster_json("geo24"))
    with pytest.raises(h.InternalError):
        h.max_flow_value(c, {"a0": (0, 12), "a1": (12, 24)})


def test_cluster_json_round_trip_and_errors():
    # test_smoke.py:28-39 (parse/serialize are host-side and in scope as I/O)
    import json
    import paper_2406_01566_b200 as h
    text = json.dumps({
        "model": {"name": "tiny", "num_layers": 4, "param_gb": 4},
        "coordinator": {"id": "coord"},
        "nodes": [{"id": "a", "vram_gb": 9, "peak_layer_tokens_per_s": 1200},
                  {"id": "b", "vram_gb": 9, "peak_layer_tokens_per_s": 800}],
        "links": [{"src": "coord", "dst": "a", "bandwidth_mbps": 1000, "latency_ms": 1},
                  {"src": "coord", "dst": "b", "bandwidth_mbps": 1000, "latency_ms": 1},
                  {"src": "a", "dst": "coord", "bandwidth_mbps": 1000, "latency_ms": 1},
                  {"src": "b", "dst": "coord", "bandwidth_mbps": 1000, "latency_ms": 1},
                  {"src": "a", "dst": "b", "bandwidth_mbps": 1000, "latency_ms": 1}]})
    c = h.Cluster.from_json(text)
    assert c.num_layers == 4 and c.coordinator == "coord" and c.node_ids == ["a", "b"]
    again = h.Cluster.from_json(c.to_json())
    assert again.to_json() == c.to_json()
    with pytest.raises(ValueError):
        h.Cluster.from_json("{}")
    bad = json.loads(text)
    bad["nodes"][0]["bogus"] = 1
    with pytest.raises(h.ParseError):
        h.Cluster.from_json(json.dumps(bad))
    dup = json.loads(text)
    dup["links"].append(dup["links"][0])
    with pytest.raises(h.ValidationError):
        h.Cluster.from_json(json.dumps(dup))
