"""Randomised GPU-vs-oracle sweep (robustness evidence beyond tests/): random
cluster sizes, interconnect densities, link bandwidths and capacity modes; chain,
uniform, link-walk and replicated-stage placements; partial and strict; both
modes.  PARITY must be bit-identical to the oracle, SCORE within 1e-6 (integer
capacities: bit-identical), statuses equal.

  python tools/fuzz_parity.py [--seconds 300] [--seed 1]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2406_01566_b200 as h  # noqa: E402
from paper_2406_01566_b200 import clusters  # noqa: E402
from _support import Oracle  # noqa: E402  (test infrastructure: the checker)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def random_cluster(rng):
    n = int(rng.choice([8, 16, 24, 31, 40, 47, 63, 64, 65, 80, 100, 130, 200]))
    peers = 0 if n <= 64 and rng.random() < 0.5 else int(rng.integers(2, 14))
    cap = "int" if rng.random() < 0.4 else "float"
    model = "llama-30b" if n < 40 else "llama2-70b"
    d = clusters.mesh_cluster(n, model=model, capacity=cap, peers=peers, seed=int(rng.integers(1, 1 << 30)))
    if rng.random() < 0.3:  # slow links: the interconnect, not compute, binds
        for l in d["links"]:
            if l["src"] != "coord" and l["dst"] != "coord":
                l["bandwidth_mbps"] = float(rng.choice([12.0, 100.0, 1000.0]))
    return d, cap


def placements(rng, e, c, n, N):
    kmax = list(e.kmax)
    L = c.num_layers
    kinds = []
    rows = [h.generate_host(kmax, L, int(rng.integers(1 << 30)), 0, n // 4, 0)]
    kinds.append("chain")
    rows.append(h.generate_host(kmax, L, int(rng.integers(1 << 30)), 0, n // 4, int(rng.integers(100000, 1000001))))
    kinds.append("uniform-mix")
    rows.append(e.generate_walk_host(int(rng.integers(1 << 30)), 0, n // 4))
    kinds.append("walk")
    rep = np.zeros((n // 4, N, 2), np.int16)  # replicated stages (dense graphs)
    for b in range(n // 4):
        groups = int(rng.integers(2, 9))
        span = max(1, min(kmax) if min(kmax) > 0 else 1)
        for k in range(N):
            g = k % groups
            s = min(g * span, L - 1)
            rep[b, k] = (s, min(s + span, L)) if kmax[k] >= span else (0, 0)
    rows.append(rep)
    kinds.append("replicated")
    return np.concatenate(rows).astype(np.int16), kinds


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--per-cluster", type=int, default=2000)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    stats = {"clusters": 0, "candidates": 0, "nonzero": 0, "status_nonzero": 0, "failures": []}
    while time.time() - t0 < a.seconds:
        d, cap = random_cluster(rng)
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c)
        o = Oracle(d)
        N = len(d["nodes"])
        rows, _ = placements(rng, e, c, a.per_cluster, N)
        for partial in (True, False):
            want_v, want_s = o.score(rows, partial)
            e.mode = "parity"
            v, s = e.score(rows, partial)
            ok_p = np.array_equal(s, want_s) and np.array_equal(bits(v), bits(want_v))
            e.mode = "score"
            vs_, ss_ = e.score(rows, partial)
            if cap == "int":
                ok_s = np.array_equal(ss_, want_s) and np.array_equal(bits(vs_), bits(want_v))
            else:
                ok_s = np.array_equal(ss_, want_s) and bool(
                    np.all(np.abs(vs_ - want_v) <= 1e-6 * np.maximum(1.0, np.abs(want_v))))
            stats["candidates"] += len(rows)
            stats["nonzero"] += int((want_v > 0).sum())
            stats["status_nonzero"] += int((want_s != 0).sum())
            if not (ok_p and ok_s):
                bad = np.nonzero((s != want_s) | (bits(v) != bits(want_v)) | (ss_ != want_s))[0][:5]
                stats["failures"].append({"n": N, "links": len(d["links"]), "cap": cap, "partial": partial,
                                          "parity_ok": bool(ok_p), "score_ok": bool(ok_s),
                                          "rows": bad.tolist()})
        stats["clusters"] += 1
    stats["seconds"] = time.time() - t0
    print(json.dumps(stats))
    return 1 if stats["failures"] else 0


if __name__ == "__main__":
    sys.exit(main())
