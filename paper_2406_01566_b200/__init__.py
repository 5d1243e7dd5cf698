"""B200-native drop-in for Helix's placement-scoring hot path.

Mirrors the reference's Python package (proj/python/helio/__init__.py) for the
hot-path surface — ``Cluster``, ``Plan``, ``max_flow_value``,
``plan_for_placement``, ``ParseError``/``ValidationError`` — and adds the
batched entry points of the B200 engine:

* ``Engine(cluster, device)``: ``score`` (host arrays, copies inside),
  ``score_device`` (device pointers), ``flows`` (per-edge flows in reference
  edge order), ``route`` (IWRR routes), ``generate_device``, ``argmax_device``;
* ``max_flow_values`` / ``best_placement`` / ``route_requests`` helpers;
* placement search: ``heuristic_placement`` (swarm / petals / sp, the
  reference's heuristics.cpp), ``local_search`` and ``plan(cluster, "local")``
  (device best-improvement search seeded from those heuristics),
  ``Engine.best_exhaustive``.

Every result is computed by the CUDA kernels in ``csrc/`` (sm_100a).  There is
no CPU fallback: importing fails loudly if the extension is missing, and using
it without a B200 raises ``InternalError``.
"""

from __future__ import annotations

import os

try:
    from . import _helio  # noqa: F401
except ImportError as exc:  # pragma: no cover - exercised only on broken installs
    raise ImportError(
        "paper_2406_01566_b200: the native extension (_helio, lib/libhelio_gpu.so) is not built; "
        "run `python -c 'import __graft_entry__ as g; g.build()'` — there is no CPU fallback"
    ) from exc

from ._helio import (  # noqa: E402
    Cluster,
    Engine,
    FlowGraph,
    InternalError,
    IwrrPicker,
    MultiEngine,
    NcclComm,
    ParseError,
    Plan,
    Scheduler,
    ValidationError,
    build_flow_graph,
    generate_host,
    generate_trace,
    generate_trace_arrays,
    heuristic_placement,
    iwrr_weights,
    local_search,
    max_flow,
    max_flow_raw,
    max_flow_value,
    nccl_unique_id,
    plan,
    plan_for_placement,
    prune_links,
    route_requests,
    simulate,
    throughput_upper_bound,
)

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")


def placement_rows(cluster, placements):
    """{node_id: (start, end)} dicts -> int16 (B, N, 2) rows in declared node order."""
    import numpy as np

    ids = cluster.node_ids
    pos = {nid: i for i, nid in enumerate(ids)}
    out = np.zeros((len(placements), len(ids), 2), dtype=np.int16)
    for b, p in enumerate(placements):
        for nid, (s, e) in p.items():
            if nid not in pos:
                raise ValidationError(f"placement references unknown node '{nid}'")
            out[b, pos[nid]] = (s, e)
    return out


def max_flow_values(cluster, placements, allow_partial=True, engine=None):
    """Batched build_flow_graph + max_flow: (values float64[B], status int32[B])."""
    eng = engine if engine is not None else Engine(cluster)
    return eng.score(placements, allow_partial)


def best_placement(cluster, placements, allow_partial=True, engine=None):
    """(value, index) of the first maximum over status-OK candidates with value > 0
    (tests/oracles/enumerate.hpp:59); (0.0, -1) if none."""
    import numpy as np

    vals, st = max_flow_values(cluster, placements, allow_partial, engine)
    ok = (st == 0) & (vals > 0)
    if not ok.any():
        return 0.0, -1
    masked = np.where(ok, vals, -1.0)
    i = int(np.argmax(masked))
    return float(vals[i]), i


__all__ = [
    "Cluster", "Engine", "FlowGraph", "InternalError", "IwrrPicker", "ParseError", "Plan",
    "ValidationError", "best_placement", "build_flow_graph", "generate_host", "generate_trace",
    "iwrr_weights", "max_flow", "max_flow_raw", "max_flow_value", "max_flow_values",
    "placement_rows", "plan_for_placement", "route_requests", "heuristic_placement", "local_search",
    "plan", "Scheduler", "simulate", "prune_links", "throughput_upper_bound", "generate_trace_arrays",
    "MultiEngine", "NcclComm", "nccl_unique_id",
]
