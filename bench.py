#!/usr/bin/env python
"""Benchmark: max-flow placement evals/sec on the 42-node LLaMA-2-70B cluster.

One step = score one batch of candidate placements (build each placement's
flow network + solve its max-flow, K1+K2) and reduce the best placement
(K4 argmax; on N>1 ranks one 16-byte NCCL all-gather of the per-rank records).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Weak scaling: every rank scores its own 1,000,000 candidates of the global
batch (global index range [r*1M, (r+1)*1M), generated on device by the
counter-based G(seed, i) before timing).  `value` is device-timed (CUDA events
on the launching stream, max over ranks); `e2e` goes through the C ABI's
host-buffer entry (helio_gpu_score_host: H2D of the placements, kernels, D2H of
every value + status) timed on the host.  --impl reference times the
unmodified reference (oracle/_ref/libhelio_ref.so, compiled from
/root/reference) on the host cores with every hardware thread.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max-flow placement evals/sec (42-node LLaMA-2-70B graph) at 1/2/4/8 B200"
WORKLOAD = ("het42-70b: covering-chain placements (SURVEY.md §8(d) G(seed,i)) on 42 nodes "
            "(4 A100-40, 6 V100-16, 8 L4-24, 10 T4-16, 4 2xL4, 6 2xT4, 4 4xT4), full mesh "
            "10 Gb/s (1,806 links), LLaMA-2-70B (80 layers), allow_partial=true")
SEED = 20240611
# --config other than the headline: the BASELINE configs as extra bench lines
# (sparse topologies draw link-walking placements)
WALK_CONFIGS = {"syn256-120l", "geo24-70b"}


def workload_of(name):
    if name == "het42-70b":
        return WORKLOAD
    gen = "link-walking" if name in WALK_CONFIGS else "covering-chain"
    return f"{name}: {gen} placements (SURVEY.md §8(d)), paper_2406_01566_b200.clusters.{name}, allow_partial=true"


def host_rows(h, name, kmax, L, first, n, ppm=0, eng=None):
    """Candidate rows on the host: G(seed, i) chains, or link walks (which need
    the compiled cluster's link lists, i.e. an engine)."""
    if name in WALK_CONFIGS:
        return eng.generate_walk_host(SEED, first, n)
    return h.generate_host(kmax, L, SEED, first, n, ppm)


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# committed ncu --set full captures of one score_kernel launch (tools/profile_score.py):
# (config, mode) -> (file under profiles/, candidates in the profiled launch)
PROFILES = {
    ("het42-70b", "score"): ("r01_score_mode_raw.csv", 200_000),
    ("het42-70b", "parity"): ("r01_parity_mode_raw.csv", 200_000),
    ("syn256-120l", "score"): ("r01_syn256_score_raw.csv", 20_000),
}


def _profile(config, mode):
    f, n = PROFILES.get((config, mode), (None, 0))
    return (os.path.join(ROOT, "profiles", f), n) if f else (None, 0)


def ncu_traffic_per_eval(config, mode):
    """DRAM bytes (read + write) per candidate of the committed ncu --set full
    capture of score_kernel for this config and mode (PROFILES)."""
    import csv
    path, graphs = _profile(config, mode)
    if path is None:
        return None, None, 0
    try:
        rows = list(csv.reader(open(path)))
        h, u, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(name)
            tot += float(v[i].replace(",", "")) * scale.get(u[i], 1.0)
        return tot / graphs, os.path.relpath(path, ROOT), graphs
    except Exception:
        return None, None, 0


def ncu_inst_per_eval(config, mode):
    """Warp-instructions per candidate (smsp__inst_executed.sum) of the same
    committed capture."""
    import csv
    path, graphs = _profile(config, mode)
    if path is None:
        return None
    try:
        rows = list(csv.reader(open(path)))
        i = rows[0].index("smsp__inst_executed.sum")
        return float(rows[2][i].replace(",", "")) / graphs
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            # nvidia-smi takes a moment to start: wait for its first sample so a
            # short timed region (e.g. 5 syn256 steps) is still covered
            t0 = time.time()
            while time.time() - t0 < 5.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def reference_rate(cluster_dict, kmax, L, budget_s, threads, first=0, rows_fn=None):
    """The unmodified reference (oracle/_ref) on the host cores: build_flow_graph
    + max_flow per candidate on a std::thread pool.  Returns (evals/s, sample).
    Inputs are prepared outside the timed call (rows_fn(first, n), default
    G(seed, i) chains)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _support import RefCluster, ref_available  # test infrastructure: reference arm only
    import paper_2406_01566_b200 as h

    if not ref_available():
        raise RuntimeError("oracle/_ref/libhelio_ref.so missing (build in the container with /root/reference)")
    if rows_fn is None:
        rows_fn = lambda f, n: h.generate_host(kmax, L, SEED, f, n, 0)  # noqa: E731
    rc = RefCluster(cluster_dict)
    probe = rows_fn(first, 64 * threads)
    t0 = time.perf_counter()
    rc.score(probe, True, threads)
    rate = len(probe) / max(time.perf_counter() - t0, 1e-6)
    n = int(min(max(rate * budget_s, 64 * threads), 400_000))
    rows = rows_fn(first, n)
    t0 = time.perf_counter()
    rc.score(rows, True, threads)
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def routing_leg(h, clusters, dev, sp, requests, with_reference):
    """configs[3]: geo24 placement scoring + IWRR routing of 1M requests.
    Score 100k candidates (SCORE), take the first-max plan, materialise its
    flows (PARITY, plan_from_placement's filter), route `requests` requests of
    generate_trace(seed 7) in the AC8 admit/complete order on the device, and
    time the reference's sequential Scheduler on the same plan and requests."""
    import numpy as np
    import torch

    d = clusters.CONFIGS["geo24"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c, device=dev)
    e.mode = "score"
    B = 100_000
    pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device=f"cuda:{dev}")
    e.generate_device(SEED, 0, B, 0, pl.data_ptr(), sp)
    v = torch.empty(B, dtype=torch.float64, device=pl.device)
    st = torch.empty(B, dtype=torch.int32, device=pl.device)
    bv = torch.empty(1, dtype=torch.float64, device=pl.device)
    bi = torch.empty(1, dtype=torch.int64, device=pl.device)
    e.score_device(pl.data_ptr(), B, v.data_ptr(), st.data_ptr(), True, sp)
    e.argmax_device(v.data_ptr(), st.data_ptr(), B, 0, bv.data_ptr(), bi.data_ptr(), sp)
    torch.cuda.synchronize(pl.device)
    row = pl[int(bi.item())].cpu().numpy()
    pe, pf, obj = e.plan_edges(row)
    _, inl, outl = h.generate_trace(requests, 0.0, "offline", 7)
    e.route(row, pe, pf, inl[:1000], outl[:1000], 0, False)  # warm-up
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        nh, hn, _, _, den = e.route(row, pe, pf, inl, outl, 0, False)  # max_hops: the plan's longest route
        times.append(time.perf_counter() - t0)
    H = hn.shape[1]
    rate = requests / min(times)
    out = {"workload": f"geo24 (acceptance geo24(), 3 regions, 12 Mb/s WAN): best of {B} candidates "
                       f"(value {float(bv.item()):.3f}), plan_from_placement, IWRR routes of "
                       f"generate_trace({requests}, offline, seed 7) in AC8 order",
           "requests": requests, "value": rate, "unit": "routes/s",
           "timing": "host wall clock around helio_gpu_route_host (H2D lengths, kernels, D2H hop nodes)",
           "hops_mean": float(nh[nh > 0].mean()), "deferred": int(den), "plan_edges": int(len(pf))}
    if with_reference:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from _support import RefCluster  # test infrastructure: reference timing only
            rc = RefCluster(d)
            t0 = time.perf_counter()
            rden, rnh, rhn, _, _ = rc.route(row, inl, outl, True, seed=7)
            rt = time.perf_counter() - t0
            m = np.arange(H)[None, :] < np.maximum(nh, 0)[:, None]
            same = bool(rden == den and np.array_equal(rnh, nh) and int(nh.max()) <= H
                        and np.array_equal(rhn[:, :H][m], hn[m]))
            out["reference"] = {"value": requests / rt, "unit": "routes/s", "cores": 1,
                                "kind": "reference", "sample": f"{requests} Scheduler::admit+complete, one thread"}
            out["identical_to_reference"] = same
        except Exception as ex:
            out["reference"] = {"value": None, "sample": f"unavailable: {ex}"}
    return out


OTHER_CONFIGS = [
    # (config, capacity, generator, candidates) — BASELINE.json configs[0,1,3,4]; het42 int-capacity
    ("single24-70b", "float", "chain", 100_000),
    ("single24-30b", "float", "chain", 100_000),
    ("geo24", "float", "chain", 100_000),
    ("het42-70b", "int", "chain", 100_000),
    ("syn256-120l", "float", "walk", 20_000),
]


def config_table(h, clusters, dev, sp, with_reference):
    """Throughput of both modes on the other BASELINE configs (parity-test
    cases of the tier; reported for coverage, not the headline)."""
    import numpy as np
    import torch

    rows = []
    for name, cap, gen, B in OTHER_CONFIGS:
        d = clusters.CONFIGS[name](cap)
        c = h.Cluster.from_json(json.dumps(d))
        e = h.Engine(c, device=dev)
        pl = torch.empty((B, e.num_nodes, 2), dtype=torch.int16, device=f"cuda:{dev}")
        if gen == "walk":
            e.generate_walk_device(SEED, 0, B, pl.data_ptr(), sp)
        else:
            e.generate_device(SEED, 0, B, 0, pl.data_ptr(), sp)
        v = torch.empty(B, dtype=torch.float64, device=pl.device)
        st = torch.empty(B, dtype=torch.int32, device=pl.device)
        rec = {"config": name, "capacity": cap, "generator": gen, "candidates": B,
               "nodes": e.num_nodes, "links": c.num_links, "layers": c.num_layers}
        out_vals = {}
        for mode in ("score", "parity"):
            e.mode = mode
            for _ in range(2):
                e.score_device(pl.data_ptr(), B, v.data_ptr(), st.data_ptr(), True, sp)
            ms = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(torch.cuda.current_stream(pl.device))
                e.score_device(pl.data_ptr(), B, v.data_ptr(), st.data_ptr(), True, sp)
                b.record(torch.cuda.current_stream(pl.device))
                torch.cuda.synchronize(pl.device)
                ms.append(a.elapsed_time(b))
            rec[mode] = B / (min(ms) / 1e3)
            out_vals[mode] = v.cpu().numpy().copy()
        e.mode = "parity"
        rec["nonzero_fraction"] = float((out_vals["parity"] > 0).mean())
        rel = np.abs(out_vals["score"] - out_vals["parity"]) / np.maximum(1.0, np.abs(out_vals["parity"]))
        rec["score_vs_parity_max_rel"] = float(rel.max())
        if with_reference:
            try:
                sys.path.insert(0, os.path.join(ROOT, "tests"))
                from _support import RefCluster  # test infrastructure: reference timing only
                rc = RefCluster(d)
                threads = os.cpu_count() or 1
                n = min(B, 200 * threads if e.num_nodes > 100 else 2000 * threads)
                host_rows = pl[:n].cpu().numpy()
                t0 = time.perf_counter()
                rv, _ = rc.score(host_rows, True, threads)
                rec["reference"] = {"value": n / (time.perf_counter() - t0), "cores": threads,
                                    "kind": "reference", "sample": f"first {n} candidates"}
                rec["parity_bit_exact_on_sample"] = bool(np.array_equal(
                    rv.view(np.int64), out_vals["parity"][:n].view(np.int64)))
            except Exception as ex:
                rec["reference"] = {"value": None, "sample": f"unavailable: {ex}"}
        rows.append(rec)
    return rows


def split_leg(eng, dev, sp, B=200_000):
    """The split K1 -> HBM -> K2 pipeline beside the fused kernel (PARITY), on
    the headline workload: device times, bytes through HBM, and whether the
    values are bit-identical."""
    import numpy as np
    import torch

    N = eng.num_nodes
    pl = torch.empty((B, N, 2), dtype=torch.int16, device=f"cuda:{dev}")
    eng.generate_device(SEED, 0, B, 0, pl.data_ptr(), sp)
    sb = eng.csr_slab_bytes
    slabs = torch.empty(B * sb, dtype=torch.uint8, device=pl.device)
    st = torch.empty(B, dtype=torch.int32, device=pl.device)
    v_split = torch.empty(B, dtype=torch.float64, device=pl.device)
    v_fused = torch.empty(B, dtype=torch.float64, device=pl.device)
    mode = eng.mode
    eng.mode = "parity"
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    cur = torch.cuda.current_stream(pl.device)
    for it in range(3):
        ev[0].record(cur)
        eng.build_csr_device(pl.data_ptr(), B, slabs.data_ptr(), st.data_ptr(), True, sp)
        ev[1].record(cur)
        eng.solve_csr_device(slabs.data_ptr(), B, v_split.data_ptr(), st.data_ptr(), sp)
        ev[2].record(cur)
        eng.score_device(pl.data_ptr(), B, v_fused.data_ptr(), st.data_ptr(), True, sp)
        ev[3].record(cur)
        torch.cuda.synchronize(pl.device)
    eng.mode = mode
    k1, k2, fused = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])
    eng.solve_csr_device(slabs.data_ptr(), B, v_split.data_ptr(), st.data_ptr(), sp)  # statuses of the split path
    torch.cuda.synchronize(pl.device)
    ok = st == 0  # graphs denser than the slab are refused (the fused path finishes them in its large slot)
    same = bool(torch.equal(v_split[ok].view(torch.int64), v_fused[ok].view(torch.int64)))
    return {"candidates": B, "slab_bytes": sb, "refused_fraction": float((~ok).float().mean().item()),
            "k1_build_ms": k1, "k2_solve_ms": k2, "fused_ms": fused,
            "split_evals_per_s": B / ((k1 + k2) / 1e3), "fused_evals_per_s": B / (fused / 1e3),
            "k1_write_gbs": B * sb / (k1 / 1e3) / 1e9, "k2_read_gbs": B * sb / (k2 / 1e3) / 1e9,
            "bit_identical_to_fused": same}


def search_leg(h, clusters, dev):
    """device local search (helio_gpu_local_search)
    on het42-70b from the reference's three heuristics, single-node moves with
    and without interval swaps, both modes; best-of-three host wall clock
    around each call (neighbour generation, scoring, argmax and the per-move
    readback all inside)."""
    import numpy as np

    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    eng = h.Engine(c, dev)
    N = eng.num_nodes
    singles = sum(1 + sum(min(c.num_layers, s + k) - s for s in range(c.num_layers)) for k in eng.kmax)
    out = {"workload": "het42-70b: best-improvement local search from swarm / petals / sp seeds",
           "neighbourhood": {"single_node_moves": singles, "interval_swaps": N * (N - 1) // 2},
           "runs": []}
    for method in ("swarm", "petals", "sp"):
        placement, _ = h.heuristic_placement(c, method)
        seed = h.placement_rows(c, [{k: tuple(v) for k, v in placement.items()}])[0]
        for mode, swaps in (("score", False), ("score", True), ("parity", True)):
            eng.mode = mode
            eng.local_search(seed, True, 1, swaps)  # warm (allocations, first launch)
            dt = float("inf")
            for _ in range(3):  # best of three (host wall clock)
                t0 = time.perf_counter()
                value, row, moves, scored = eng.local_search(seed, True, -1, swaps)
                dt = min(dt, time.perf_counter() - t0)
            v0, _ = eng.score(seed[None])
            out["runs"].append({"seed": method, "mode": mode, "swaps": swaps, "seed_value": float(v0[0]),
                                "value": value, "moves": moves, "scored": scored, "seconds": dt,
                                "evals_per_s": scored / dt if dt > 0 else None})
    # past the local optimum: sampled multi-node search (helio_gpu_sampled_search)
    # from the petals seed's local optimum, then one more local search
    eng.mode = "score"
    placement, _ = h.heuristic_placement(c, "petals")
    seed = h.placement_rows(c, [{k: tuple(v) for k, v in placement.items()}])[0]
    lv, lrow, _, _ = eng.local_search(seed)
    rounds, batch, changes = 10, 1 << 20, 2
    t0 = time.perf_counter()
    sv, srow, imp, sscored = eng.sampled_search(lrow, True, rounds, batch, changes, 7)
    dt = time.perf_counter() - t0
    fv, _, fmoves, _ = eng.local_search(srow)
    out["sampled"] = {"from": "petals local optimum", "mode": "score", "rounds": rounds, "batch": batch,
                      "max_changes": changes, "start_value": lv, "value": sv, "improving_rounds": imp,
                      "scored": sscored, "seconds": dt, "evals_per_s": sscored / dt if dt > 0 else None,
                      "local_search_after": fv,
                      "note": "petals-derived mutants carry ~5N edges: they run in the middle slot tier"}
    return out


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import paper_2406_01566_b200 as h
    from paper_2406_01566_b200 import clusters

    d = clusters.CONFIGS[args.config]("float")
    c = h.Cluster.from_json(json.dumps(d))
    kmax = [c.max_layers(i) for i in c.node_ids]
    threads = os.cpu_count() or 1
    rows_fn = None
    if args.config in WALK_CONFIGS:  # link walks need the compiled link lists (input prep, untimed)
        gen = h.Engine(c)
        rows_fn = lambda f, n: host_rows(h, args.config, kmax, c.num_layers, f, n, eng=gen)  # noqa: E731
    rates = []
    samples = 0
    step_ms = []
    for step in range(args.warmup + args.steps):
        r, n, dt = reference_rate(d, kmax, c.num_layers, args.ref_step_s, threads, first=step * 10_000_000,
                                  rows_fn=rows_fn)
        if step >= args.warmup:
            rates.append(r)
            samples += n
            step_ms.append(n / r * 1e3 if r else None)
    value = sorted(rates)[len(rates) // 2]
    ms = [x for x in step_ms if x]
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(ms) / len(ms) if ms else None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_of(args.config), "parallelism": "host threads",
                   "candidates_per_step": samples // max(1, args.steps)},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "reference",
                         "sample": f"median of {args.steps} steps, each ~{args.ref_step_s:.0f}s of "
                                   f"build_flow_graph+max_flow on the first candidates of the workload "
                                   f"(std::thread pool, {threads} threads)"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="het42-70b")
    ap.add_argument("--per-gpu", type=int, default=1_000_000)
    ap.add_argument("--ppm", type=int, default=0, help="uniform-interval mix, parts per million")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-routing", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--route-requests", type=int, default=1_000_000)
    ap.add_argument("--mode", default="score", choices=["score", "parity"],
                    help="headline scoring mode (the other mode is timed too and reported beside it)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_01566_b200 as h
    from paper_2406_01566_b200 import clusters

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    d = clusters.CONFIGS[args.config]("float")
    c = h.Cluster.from_json(json.dumps(d))
    eng = h.Engine(c, device=local)
    eng.mode = args.mode
    N, L = eng.num_nodes, eng.num_layers
    B = args.per_gpu
    first = rank * B
    # a dedicated stream: its handle is what the engine launches on, and the
    # CUDA events below are recorded on the same stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream

    pl = torch.empty((B, N, 2), dtype=torch.int16, device=dev)
    if args.config in WALK_CONFIGS:
        eng.generate_walk_device(SEED, first, B, pl.data_ptr(), sp)
    else:
        eng.generate_device(SEED, first, B, args.ppm, pl.data_ptr(), sp)
    vals = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    best = torch.empty(1, dtype=torch.float64, device=dev)
    bidx = torch.empty(1, dtype=torch.int64, device=dev)
    rec = torch.empty(2, dtype=torch.int64, device=dev)
    gathered = torch.empty(2 * world, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def step():
        eng.score_device(pl.data_ptr(), B, vals.data_ptr(), st.data_ptr(), True, sp)
        eng.argmax_device(vals.data_ptr(), st.data_ptr(), B, first, best.data_ptr(), bidx.data_ptr(), sp)
        if world > 1:
            rec[0:1].copy_(best.view(torch.int64))
            rec[1:2].copy_(bidx)
            dist.all_gather_into_tensor(gathered, rec)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches0 = eng.launch_count
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            kernel_ms.append(eng.last_kernel_ms())
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    launches = eng.launch_count - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = (B * world) / (ms_per_step / 1e3)

    # the other mode, same batch, same timing rules (reported beside the headline)
    other = "parity" if args.mode == "score" else "score"
    eng.mode = other
    oth = []
    for i in range(args.steps + 1):
        flush.zero_()
        a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b2.record(stream)
        torch.cuda.synchronize(dev)
        if i > 0:
            oth.append(a.elapsed_time(b2))
    eng.mode = args.mode
    ot = torch.tensor([sum(oth)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ot, op=dist.ReduceOp.MAX)
    other_rate = (B * world) / (float(ot.item()) / len(oth) / 1e3)
    eng.mode = other
    step()
    torch.cuda.synchronize(dev)
    other_vals = vals.clone()
    eng.mode = args.mode
    step()
    torch.cuda.synchronize(dev)
    rel = ((vals - other_vals).abs() / other_vals.abs().clamp(min=1.0)).max().item()

    # winner (deterministic: max value, then min global index)
    from paper_2406_01566_b200.dist import reduce_best, unpack_records
    recs = unpack_records(gathered) if world > 1 else [(float(best.item()), int(bidx.item()))]
    win = reduce_best(recs)
    # the winner's plan reaches every rank: its owner
    # computes the PARITY per-edge flows and broadcasts row + flows over NCCL
    winner_plan = None
    if world > 1 and win[1] >= 0:
        from paper_2406_01566_b200.dist import share_winner
        row_w = flows_w = None
        if win[1] // B == rank:
            row_w = pl[win[1] - first].cpu().numpy()
            _, _, _, ne_w, _, dbl_w = eng.flows(row_w[None], True)
            flows_w = dbl_w[0, :int(ne_w[0]), 1]
        t_share = time.perf_counter()
        row_s, flows_s = share_winner(win[1], B, row_w, flows_w)
        winner_plan = {"owner_rank": win[1] // B, "edges": int(flows_s.size),
                       "bytes": int(row_s.nbytes + flows_s.nbytes),
                       "ms": (time.perf_counter() - t_share) * 1e3}
    st_host = st.cpu().numpy()
    nonzero = float((vals.cpu().numpy() > 0).mean())

    # roofline of the dominant kernel (fused build+solve): algorithmic bytes per
    # eval = 4N (int16 start/end in) + 8 (value) + 4 (status) — SURVEY §8(d).
    bytes_per_eval = 4 * N + 8 + 4
    kms = [k for k in kernel_ms if k and k > 0]
    avg_kernel_ms = sum(kms) / len(kms) if kms else ms_per_step
    achieved = bytes_per_eval * B / (avg_kernel_ms / 1e3) / 1e9
    peak, peak_src = load_peaks()
    tpe, tsrc, tgraphs = ncu_traffic_per_eval(args.config, args.mode)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": (tpe * B) if tpe is not None else None,
                "traffic_unit": "bytes per launch (DRAM read + write)",
                "traffic_source": (f"{tsrc}: ncu --set full of one {tgraphs}-candidate launch, per candidate x {B}"
                                   if tsrc else "no committed capture for this config/mode"),
                "algorithmic_bytes_per_launch": bytes_per_eval * B,
                "kernel": f"score_kernel<{args.mode}> (fused K1 build + K2 solve, one warp per graph)",
                "kernel_ms": avg_kernel_ms, "kernel_share_of_step": avg_kernel_ms / ms_per_step,
                "bytes_per_eval": bytes_per_eval, "peak_source": peak_src,
                "note": "latency/issue-bound SIMT graph kernel: HBM fraction is structurally tiny; "
                        "see DESIGN.md and profiles/ for issue/smem evidence"}

    # e2e through the C ABI with host buffers (pinned), timed on the host
    e2e = None
    if not args.no_e2e:
        host = torch.from_numpy(host_rows(h, args.config, list(eng.kmax), L, first, B, args.ppm, eng)).pin_memory()
        hv = torch.empty(B, dtype=torch.float64).pin_memory()
        hs = torch.empty(B, dtype=torch.int32).pin_memory()
        for _ in range(2):
            eng.score_best_host_ptr(host.data_ptr(), B, hv.data_ptr(), hs.data_ptr(), True)
        times = []
        for _ in range(args.steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_best = eng.score_best_host_ptr(host.data_ptr(), B, hv.data_ptr(), hs.data_ptr(), True)
            times.append(time.perf_counter() - t0)
        if world == 1:
            assert int(e2e_best[1]) == recs[0][1], "e2e winner differs from the device path"
        tt = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_rate = B * world * args.steps / float(tt.item())
        assert torch.equal(hv.view(torch.int64), vals.cpu().view(torch.int64)), "e2e values differ from device path"
        e2e = {"value": e2e_rate, "unit": "evals/s", "h2d_bytes_per_step": B * world * 4 * N,
               "d2h_bytes_per_step": B * world * 12 + 16 * world,
               "call": "helio_gpu_score_best_host (pinned host placements in; every value + status and the "
                       "first-max winner out)"}

    # extras (single-GPU views) only at N = 1: at N > 1 the other ranks must not
    # wait on rank 0 outside the timed region
    split = None
    if world == 1 and not args.no_configs:
        try:
            split = split_leg(eng, local, sp)
        except Exception as ex:  # reported, never fatal
            split = {"error": str(ex)}

    cfg_table = None
    if world == 1 and not args.no_configs:
        try:
            cfg_table = config_table(h, clusters, local, sp, with_reference=(world == 1 and not args.no_cpu_baseline))
        except Exception as ex:  # reported, never fatal
            cfg_table = [{"error": str(ex)}]

    routing = None
    if world == 1 and not args.no_routing:
        try:
            routing = routing_leg(h, clusters, local, sp, args.route_requests,
                                  with_reference=(world == 1 and not args.no_cpu_baseline))
        except Exception as ex:  # reported, never fatal
            routing = {"value": None, "error": str(ex)}

    search = None
    if world == 1 and not args.no_configs:
        try:
            search = search_leg(h, clusters, local)
        except Exception as ex:  # reported, never fatal
            search = {"error": str(ex)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            r, n, dt = reference_rate(d, list(eng.kmax), L, args.cpu_seconds, threads,
                                      rows_fn=lambda f, n: host_rows(h, args.config, list(eng.kmax), L, f, n,
                                                                     eng=eng))
            cpu = {"value": r, "unit": "evals/s", "cores": threads, "kind": "reference",
                   "sample": f"first {n} candidates of the workload, {dt:.1f}s wall, unmodified reference "
                             f"build_flow_graph+max_flow on a {threads}-thread std::thread pool"}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "evals/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {ex}"}

    if search and cpu and cpu.get("value") and "runs" in search:
        for r in search["runs"]:  # the same scoring on the reference, at the measured host rate
            r["reference_equivalent_seconds"] = r["scored"] / cpu["value"]

    clocks = clk.summary()
    if world > 1:  # every rank sampled its own GPU: report them all (the step is as slow as the slowest)
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"sm_mhz": clocks.get("sm_mhz"), "reasons": clocks.get("reasons"),
                                          "kernel_ms": sum(k for k in kernel_ms if k) / max(1, len(kernel_ms))})
        clocks["per_rank"] = per_rank
    # the roofline that binds this kernel: warp-instruction issue (4 schedulers
    # per SM, one instruction per clock each) — see DESIGN.md §4
    ipe = ncu_inst_per_eval(args.config, args.mode)
    if ipe and clocks.get("sm_mhz"):
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        issue_peak = sms * 4 * clocks["sm_mhz"] * 1e6
        issue_ach = ipe * B / (avg_kernel_ms / 1e3)
        roofline["issue"] = {"bound": "warp-instruction issue", "warp_instr_per_eval": ipe,
                             "achieved": issue_ach, "peak": issue_peak, "unit": "warp-instr/s",
                             "frac": issue_ach / issue_peak,
                             "source": "smsp__inst_executed.sum per candidate from the committed ncu capture; "
                                       "peak = SMs x 4 schedulers x median SM clock under load"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_of(args.config), "candidates_per_gpu": B, "global_batch": B * world,
                       "parallelism": f"dp{world} (candidate shards; NCCL all-gather of the 16 B argmax record)",
                       "mode": args.mode, "p_uniform_ppm": args.ppm,
                       "other_mode": {"mode": other, "value": other_rate, "unit": "evals/s",
                                      "max_rel_diff_vs_headline": rel},
                       "l2": "L2 flushed (256 MB write) between timed steps; inputs 168 MB/GPU",
                       "nonzero_fraction": nonzero, "status_nonzero": int((st_host != 0).sum()),
                       "best": {"value": win[0], "index": win[1]}, "winner_plan_broadcast": winner_plan},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "routing": routing, "other_configs": cfg_table, "split_pipeline": split, "search": search,
            "clocks": clocks,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
