"""Randomised masked-routing sweep against the reference (robustness evidence
beyond tests/): random mesh clusters (full or sparse, int or float capacities),
plans from good sampled placements (partial or strict), KV sizes drawn over four
decades so 0-100% of admissions are deferred, random traces; every request's
hop count, deferral and hop nodes / exec ranges must equal the reference's
Scheduler::admit/complete replay (oracle/_ref).  Each case runs the default
replay and, at random, the exact-passes-only variant or the serial warp kernel.

  python tools/fuzz_routing.py [--seconds 300] [--seed 1]
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
from _support import RefCluster  # noqa: E402  (test infrastructure: the checker)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    st = {"cases": 0, "requests": 0, "deferred": 0, "by_variant": {}, "deferral_fractions": [], "failures": []}
    while time.time() - t0 < a.seconds:
        n = int(rng.choice([6, 8, 12, 16, 24, 31, 42, 48, 64]))
        peers = 0 if rng.random() < 0.5 else int(rng.integers(2, 8))
        cap = "int" if rng.random() < 0.3 else "float"
        d = clusters.mesh_cluster(n, model="llama2-70b" if n >= 24 else "llama-30b", capacity=cap, peers=peers,
                                  seed=int(rng.integers(1, 1 << 30)))
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c)
        e.mode = "score"
        rows = h.generate_host(list(e.kmax), c.num_layers, int(rng.integers(1 << 30)), 0, 4000,
                               int(rng.choice([0, 200000])))
        v, s = e.score(rows)
        ok = np.nonzero((s == 0) & (v > 0))[0]
        if len(ok) == 0:
            continue
        row = rows[ok[np.argsort(-v[ok])[int(rng.integers(0, min(len(ok), 20)))]]]
        partial = bool(rng.random() < 0.7)
        pe, pf, _ = e.plan_edges(row, partial)
        if len(pf) == 0:
            continue
        kv = float(10 ** rng.uniform(4, 7.3))
        dm = json.loads(json.dumps(d))
        dm["model"]["kv_bytes_per_token_layer"] = kv
        cm = h.Cluster.from_json(json.dumps(dm))
        em = h.Engine(cm)
        R = int(rng.choice([1000, 20000, 100000]))
        _, inl, outl = h.generate_trace_arrays(R, 0.0, "offline", int(rng.integers(1, 1 << 30)))
        variant = str(rng.choice(["default", "default", "exact_passes", "warp"]))
        os.environ.pop("HELIO_ROUTE_APPROX", None)
        os.environ.pop("HELIO_ROUTE_SPEC", None)
        if variant == "exact_passes":
            os.environ["HELIO_ROUTE_APPROX"] = "0"
        elif variant == "warp":
            os.environ["HELIO_ROUTE_SPEC"] = "0"
        try:
            nh, hn, hs, he, den = em.route(row, pe, pf, inl, outl, cm.num_layers)
        except Exception as ex:  # a ValidationError, as the reference raises
            nh = None
            err = str(ex)
        den_r, nh_r, hn_r, hs_r, he_r = RefCluster(dm).route(row, inl, outl, partial)
        case = {"n": n, "peers": peers, "cap": cap, "partial": partial, "kv": kv, "R": R, "variant": variant}
        if nh is None or den_r < 0:  # both must reject the plan
            st["rejected_both" if (nh is None and den_r < 0) else "failures"] = (
                st.get("rejected_both", 0) + 1 if (nh is None and den_r < 0)
                else st["failures"] + [{**case, "error": err if nh is None else "", "ref": int(den_r)}])
            continue
        mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
        same = (den == den_r and np.array_equal(nh, nh_r) and np.array_equal(hn[mask], hn_r[mask])
                and np.array_equal(hs[mask], hs_r[mask]) and np.array_equal(he[mask], he_r[mask]))
        st["cases"] += 1
        st["requests"] += R
        st["deferred"] += int(den_r)
        st["by_variant"][variant] = st["by_variant"].get(variant, 0) + 1
        st["deferral_fractions"].append(round(den_r / R, 3))
        if not same:
            st["failures"].append({**case, "deferred": int(den), "deferred_ref": int(den_r),
                                   "first_bad": int(np.nonzero(nh != nh_r)[0][0]) if not np.array_equal(nh, nh_r) else -1})
    fr = np.array(st["deferral_fractions"] or [0.0])
    st["deferral_fraction_quantiles"] = [float(q) for q in np.quantile(fr, [0, 0.25, 0.5, 0.75, 1])]
    del st["deferral_fractions"]
    print(json.dumps(st))
    return 1 if st["failures"] else 0


if __name__ == "__main__":
    sys.exit(main())
