"""A/B of the masked replays on the geo24 plan with KV masking binding:
route_masked_spec (chunked parallel) against route_masked_warp (serial), same
outputs required; prints routes/s of each (host wall incl. copies).
python tools/route_spec_probe.py [requests]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2406_01566_b200 as h  # noqa: E402
from _support import golden, golden_cluster  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000


def bench_plan():
    """bench.py routing_leg's plan: first max of 100k geo24 candidates."""
    import torch
    from paper_2406_01566_b200 import clusters
    c = h.Cluster.from_json(json.dumps(clusters.CONFIGS["geo24"]("float")))
    e = h.Engine(c)
    e.mode = "score"
    B = 100_000
    pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device="cuda:0")
    sp = torch.cuda.current_stream().cuda_stream
    e.generate_device(20240611, 0, B, 0, pl.data_ptr(), sp)
    v = torch.empty(B, dtype=torch.float64, device="cuda:0")
    st = torch.empty(B, dtype=torch.int32, device="cuda:0")
    bv = torch.empty(1, dtype=torch.float64, device="cuda:0")
    bi = torch.empty(1, dtype=torch.int64, device="cuda:0")
    e.score_device(pl.data_ptr(), B, v.data_ptr(), st.data_ptr(), True, sp)
    e.argmax_device(v.data_ptr(), st.data_ptr(), B, 0, bv.data_ptr(), bi.data_ptr(), sp)
    torch.cuda.synchronize()
    row = pl[int(bi.item())].cpu().numpy()
    pe, pf, _ = e.plan_edges(row)
    return clusters.CONFIGS["geo24"]("float"), row, pe, pf


def main():
    z = golden("route_geo24.npz")
    _, inl, outl = h.generate_trace_arrays(R, 0.0, "offline", 7)
    cases = []
    zpe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
    for kv in (1e6, 7e5, 2e6, 5e6):
        cases.append(("golden", kv, golden_cluster("geo24_float"), z["row"], zpe, z["plan_flow"]))
    bd, brow, bpe, bpf = bench_plan()
    for kv in (1e6, 3e6):
        cases.append(("bench", kv, bd, brow, bpe, bpf))
    for tag, kv, d0, row, pe, pf in cases:
        d = json.loads(json.dumps(d0))
        d["model"]["kv_bytes_per_token_layer"] = kv
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c)
        res = {}
        legs = (("spec", "1"),) if os.environ.get("PROBE_SPEC_ONLY") else (("warp", "0"), ("spec", "1"))
        for name, flag in legs:
            os.environ["HELIO_ROUTE_SPEC"] = flag
            best = 1e9
            for it in range(3):
                os.environ["HELIO_ROUTE_DIAG"] = "1" if it == 0 and flag == "1" else ""
                if not os.environ["HELIO_ROUTE_DIAG"]:
                    del os.environ["HELIO_ROUTE_DIAG"]
                t0 = time.perf_counter()
                out = e.route(row, pe, pf, inl, outl, 0, False)
                best = min(best, time.perf_counter() - t0)
            res[name] = (out, best)
        if "warp" not in res:
            (nh, hn, hs, he, den), ts = res["spec"]
            print(json.dumps({"plan": tag, "kv": kv, "deferred": int(den), "spec_routes_per_s": R / ts}), flush=True)
            continue
        (nh, hn, hs, he, den), tw = res["warp"]
        (nh2, hn2, hs2, he2, den2), ts = res["spec"]
        mask = np.arange(hn.shape[1])[None, :] < np.maximum(nh, 0)[:, None]
        same = den == den2 and np.array_equal(nh, nh2) and np.array_equal(hn[mask], hn2[mask])
        if not same:
            bad = np.nonzero(nh != nh2)[0]
            print("first nh mismatch", bad[:5], nh[bad[:5]], nh2[bad[:5]])
        print(json.dumps({"plan": tag, "kv": kv, "deferred": int(den), "deferred_spec": int(den2), "same": bool(same),
                          "warp_routes_per_s": R / tw, "spec_routes_per_s": R / ts}), flush=True)


if __name__ == "__main__":
    main()
