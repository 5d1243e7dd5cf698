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
WALK_CONFIGS = {"syn256-120l", "geo24-70b", "het42-70b-prune12"}


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
    ("het42-70b", "score"): ("r02_het42_score_raw.csv", 200_000),
    ("het42-70b", "parity"): ("r01_parity_mode_raw.csv", 200_000),
    ("syn256-120l", "score"): ("r02_syn256_score_raw.csv", 20_000),
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


def load_workloads():
    """The workload clusters (paper_2406_01566_b200/clusters.py: builders of
    dicts in the reference's cluster JSON schema, stdlib only) loaded by file
    path, so the reference arm never imports the package (whose import loads
    the CUDA extension)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "helio_workloads", os.path.join(ROOT, "paper_2406_01566_b200", "clusters.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class RefArm:
    """The unmodified reference (oracle/_ref/libhelio_ref.so, compiled from
    /root/reference by oracle/Makefile) through ctypes: the reference's own
    parse_cluster, ClusterSpec::max_layers, build_flow_graph + max_flow, and the
    workload generator restated over its ClusterSpec (refh_generate).  Nothing
    from paper_2406_01566_b200 is loaded on this path."""

    SO = os.path.join(ROOT, "oracle", "_ref", "libhelio_ref.so")

    def __init__(self, cluster_dict):
        import ctypes as C

        import numpy as np

        if not os.path.exists(self.SO):
            raise RuntimeError("oracle/_ref/libhelio_ref.so missing (built in the container from /root/reference)")
        self.np, self.C = np, C
        lib = C.CDLL(self.SO)
        i16 = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
        i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        f64 = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        lib.refh_cluster_from_json.restype = C.c_void_p
        lib.refh_cluster_from_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        lib.refh_cluster_free.argtypes = [C.c_void_p]
        lib.refh_cluster_num_nodes.argtypes = [C.c_void_p]
        lib.refh_max_layers.argtypes = [C.c_void_p, C.c_int]
        lib.refh_score.argtypes = [C.c_void_p, i16, C.c_int64, C.c_int, C.c_int, f64, i32]
        lib.refh_solve_only.argtypes = [C.c_void_p, i16, C.c_int64, C.c_int, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.refh_solve_only.restype = C.c_int64
        lib.refh_generate.argtypes = [C.c_void_p, C.c_uint64, C.c_int64, C.c_int64, C.c_uint32, C.c_int,
                                      C.c_int, i16]
        self.lib = lib
        err = C.create_string_buffer(512)
        self.h = lib.refh_cluster_from_json(json.dumps(cluster_dict).encode(), err, 512)
        if not self.h:
            raise RuntimeError(f"reference parse_cluster failed: {err.value.decode()}")
        self.N = lib.refh_cluster_num_nodes(self.h)
        self.kmax = [lib.refh_max_layers(self.h, k) for k in range(self.N)]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.refh_cluster_free(self.h)

    def rows(self, first, n, walk, ppm=0, threads=None):
        out = self.np.zeros((n, self.N, 2), self.np.int16)
        self.lib.refh_generate(self.h, SEED, first, n, ppm, int(walk), threads or (os.cpu_count() or 1), out)
        return out

    def score(self, rows, threads):
        n = rows.shape[0]
        v = self.np.zeros(n, self.np.float64)
        st = self.np.zeros(n, self.np.int32)
        t0 = time.perf_counter()
        self.lib.refh_score(self.h, rows, n, 1, threads, v, st)
        return v, st, time.perf_counter() - t0

    def solve_only(self, rows, threads):
        s, chk = self.C.c_double(0), self.C.c_double(0)
        g = self.lib.refh_solve_only(self.h, rows, rows.shape[0], 1, threads, self.C.byref(s), self.C.byref(chk))
        return g, s.value

    def rate(self, first, budget_s, threads, walk, ppm=0):
        """evals/s of build_flow_graph + max_flow over the workload's rows
        [first, first + n), n sized for ~budget_s; generation untimed."""
        probe = self.rows(first, 32 * threads, walk, ppm)
        for _ in range(2):  # the first call pays page faults and allocator warm-up
            _, _, dt = self.score(probe, threads)
        n = int(min(max(len(probe) / max(dt, 1e-6) * budget_s, 32 * threads), 2_000_000))
        rows = self.rows(first, n, walk, ppm)
        _, _, dt = self.score(rows, threads)
        return n / dt, n, dt


def reference_baseline(cluster_dict, walk, budget_s, ppm=0, arm=None):
    """SURVEY.md §8(d) "CPU reference timing": the unmodified reference on every
    host thread (the headline baseline), plus one core, plus max_flow alone on
    pre-built graphs, on the first candidates of the workload."""
    ra = arm or RefArm(cluster_dict)
    threads = os.cpu_count() or 1
    rate, n, dt = ra.rate(0, budget_s, threads, walk, ppm)
    r1, n1, _ = ra.rate(0, max(1.0, budget_s / 4), 1, walk, ppm)
    rows = ra.rows(0, min(n, 200_000), walk, ppm)
    g, solve_s = ra.solve_only(rows, threads)
    return {"value": rate, "unit": "evals/s", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"first {n} candidates of the workload ({dt:.1f} s wall): unmodified reference "
                      f"build_flow_graph + max_flow (enumerate.hpp:56-57) on a {threads}-thread std::thread pool",
            "single_core": {"value": r1, "unit": "evals/s", "sample": f"first {n1} candidates, 1 thread"},
            "solve_only": {"value": g / solve_s if solve_s > 0 else None, "unit": "max_flow/s",
                           "sample": f"max_flow on {g} pre-built FlowGraphs, {threads} threads"}}


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
    _, inl, outl = h.generate_trace_arrays(requests, 0.0, "offline", 7)
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
    # the stateful drop-in (Scheduler::admit / complete, one call per request,
    # picks from device-built IWRR cycles): per-admit latency in the same order
    try:
        placement = {c.node_ids[k]: (int(row[k, 0]), int(row[k, 1])) for k in range(len(row)) if row[k, 1] > row[k, 0]}
        sched = h.Scheduler(c, h.plan_for_placement(c, placement), "iwrr", 7)
        snh, secs = sched.run_ac8(inl, outl)
        out["stateful"] = {"value": requests / secs, "unit": "routes/s", "per_admit_us": secs / requests * 1e6,
                           "call": "Scheduler.admit + complete per request (AC8 order), host-timed without Python",
                           "identical_to_batch": bool(np.array_equal(snh, nh))}
    except Exception as ex:  # reported, never fatal
        out["stateful"] = {"error": str(ex)}
    # KV masking binds: the same plan with kv_bytes_per_token_layer = 1 MB
    # (3% of admissions deferred on this plan) takes the exact replay kernel
    try:
        dm = json.loads(json.dumps(d))
        dm["model"]["kv_bytes_per_token_layer"] = 1e6
        cm = h.Cluster.from_json(json.dumps(dm))
        em = h.Engine(cm, device=dev)
        em.route(row, pe, pf, inl[:1000], outl[:1000], 0, False)  # warm-up
        mt = []
        for _ in range(3):
            t0 = time.perf_counter()
            mnh, mhn, _, _, mden = em.route(row, pe, pf, inl, outl, 0, False)
            mt.append(time.perf_counter() - t0)
        out["masked"] = {"value": requests / min(mt), "unit": "routes/s", "deferred": int(mden),
                         "kernel": "route_masked_spec (exact AC8 replay: chunked speculation on the deferral set, "
                                   "wavefront over the plan DAG, one CTA)",
                         "workload": "same plan and requests, kv_bytes_per_token_layer = 1e6"}
    except Exception as ex:  # reported, never fatal
        out["masked"] = {"error": str(ex)}
    if with_reference:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from _support import RefCluster  # test infrastructure: reference timing only
            if "value" in out.get("masked", {}):
                t0 = time.perf_counter()
                rden_m, rnh_m, rhn_m, _, _ = RefCluster(dm).route(row, inl, outl, True, seed=7)
                rtm = time.perf_counter() - t0
                Hm = mhn.shape[1]
                mm = np.arange(Hm)[None, :] < np.maximum(mnh, 0)[:, None]
                out["masked"]["reference"] = {"value": requests / rtm, "unit": "routes/s", "cores": 1,
                                              "kind": "reference",
                                              "sample": f"{requests} Scheduler::admit+complete, one thread"}
                out["masked"]["identical_to_reference"] = bool(
                    rden_m == mden and np.array_equal(rnh_m, mnh) and np.array_equal(rhn_m[:, :Hm][mm], mhn[mm]))
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
    ("het42-70b-prune12", "float", "walk", 100_000),
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


# default global batch per config (BASELINE.json configs): het42 1M sharded
# over N (configs[2]), syn256 10M (configs[4]), the rest 100k (configs[1], [3])
DEFAULT_BATCH = {"het42-70b": 1_000_000, "syn256-120l": 10_000_000}


def shard(args, world, rank):
    """(first global index, candidates on this rank, global batch).  strong:
    the global batch is split into contiguous ranges [r*G/N, (r+1)*G/N);
    weak: every rank scores its own --per-gpu candidates."""
    if args.scaling == "strong":
        G = args.global_batch
        lo, hi = rank * G // world, (rank + 1) * G // world
        return lo, hi - lo, G
    return rank * args.per_gpu, args.per_gpu, args.per_gpu * world


def bench_config(args, world):
    """The `config` object — identical on both arms (static workload facts only;
    measured details live in other keys)."""
    _, n0, G = shard(args, world, 0)
    return {"workload": workload_of(args.config), "global_batch": G, "candidates_per_gpu": n0,
            "parallelism": f"dp{world} (candidate shards; NCCL all-gather of the 16 B argmax record)",
            "capacity": "float", "allow_partial": True, "generator_seed": SEED, "p_uniform_ppm": args.ppm,
            "l2": "GPU arm: L2 flushed (256 MB write) between timed steps"}


def latency_leg(h, clusters, with_reference):
    """Per-call latency of the reference-facing API (SURVEY.md §8(b) call
    sites placement.cpp:358-359, :441-442, pymodule.cpp:170-171): p50 over
    repeated single-placement calls of max_flow_value, plan_for_placement and
    build_flow_graph + max_flow on het42-70b, beside the unmodified reference
    doing the same call on one host thread; and the reference's MILP planner
    (plan_placement) at AC5's settings on geo24 (acceptance_main.cpp:371-378)
    running over this engine vs the pure reference."""
    import numpy as np

    out = {"workload": "het42-70b, the bench's first covering-chain placement; p50 of 200 calls"}
    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    eng = h.Engine(c)
    row = h.generate_host(list(eng.kmax), c.num_layers, SEED, 0, 1, 0)[0]
    placement = {c.node_ids[k]: (int(row[k, 0]), int(row[k, 1])) for k in range(len(row)) if row[k, 1] > row[k, 0]}

    def p50(fn, n=200):
        fn()
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts)) * 1e6

    def pair():
        g = h.build_flow_graph(c, placement)
        return h.max_flow(g)

    out["max_flow_value_us"] = p50(lambda: h.max_flow_value(c, placement))
    out["plan_for_placement_us"] = p50(lambda: h.plan_for_placement(c, placement))
    out["build_flow_graph_max_flow_us"] = p50(pair)
    if with_reference:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from _support import RefCluster  # test infrastructure: reference timing only
            rc = RefCluster(d)
            r1 = np.ascontiguousarray(row[None], np.int16)
            out["reference"] = {"build_flow_graph_max_flow_us": p50(lambda: rc.score(r1, True, 1)),
                                "plan_from_placement_us": p50(lambda: rc.plan(row)),
                                "cores": 1, "kind": "reference",
                                "sample": "the same placement, one host thread, via ctypes (oracle/_ref)"}
        except Exception as ex:  # reported, never fatal
            out["reference"] = {"error": str(ex)}
    # AC5: the reference's MILP over GPU scores vs the pure reference
    try:
        g = clusters.CONFIGS["geo24"]("float")
        cg = h.Cluster.from_json(json.dumps(g))
        t0 = time.perf_counter()
        p = h.plan(cg, "milp", gap=0.05, node_budget=300, prune_degree=6, lex_tiebreak=False)
        out["milp_ac5"] = {"seconds": time.perf_counter() - t0, "objective": p.objective,
                           "call": "plan(c, 'milp', gap=0.05, node_budget=300, prune_degree=6, lex_tiebreak=False): "
                                   "the reference's plan_placement linked over this engine (lib/libhelio_planner.so)"}
        if with_reference:
            from _support import RefCluster, plan_milp, ref  # test infrastructure: reference timing only
            rc = RefCluster(g)
            t0 = time.perf_counter()
            obj, _, _, _, _ = plan_milp(ref(), "refh_", rc.h, len(g["nodes"]), True, gap=0.05, lex=False,
                                        node_budget=300, prune=6.0)
            out["milp_ac5"]["reference"] = {"seconds": time.perf_counter() - t0, "objective": obj,
                                            "same_objective": bool(obj == p.objective)}
    except Exception as ex:  # reported, never fatal
        out["milp_ac5"] = {"error": str(ex)}
    return out


def run_reference(args):
    """--impl reference: the unmodified reference on the host cores, on this
    run's workload (RefArm: oracle/_ref only — no package import).  Each step
    scores a bounded sample of the global batch (rows rotate through it)."""
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", args.gpus)
    if rank != 0:
        return 0
    wl = load_workloads()
    d = wl.CONFIGS[args.config]("float")
    walk = args.config in WALK_CONFIGS
    ra = RefArm(d)
    threads = os.cpu_count() or 1
    _, _, G = shard(args, world, 0)
    # size one step for ~ref_step_s of host work (bounded: the whole run stays
    # within a few minutes), from a probe
    probe = ra.rows(0, 32 * threads, walk, args.ppm)
    for _ in range(2):  # the first call pays page faults and allocator warm-up
        _, _, dt = ra.score(probe, threads)
    n = int(min(max(len(probe) / max(dt, 1e-6) * args.ref_step_s, 32 * threads), G))
    evals, secs, step_ms = 0, 0.0, []
    for step in range(args.warmup + args.steps):
        first = (step * n) % max(1, G - n + 1)
        rows = ra.rows(first, n, walk, args.ppm)  # input preparation, untimed
        _, _, dt = ra.score(rows, threads)
        if step >= args.warmup:
            evals += n
            secs += dt
            step_ms.append(dt * 1e3)
    value = evals / secs
    base = reference_baseline(d, walk, max(2.0, args.ref_step_s), args.ppm, arm=ra)
    base.update({"value": value,
                 "sample": f"{args.steps} timed steps (+{args.warmup} warm-up) of {n} candidates each, rotating "
                           f"through the {G}-candidate workload: unmodified reference build_flow_graph + max_flow "
                           f"on a {threads}-thread std::thread pool"})
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(step_ms) / len(step_ms), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out))
    return 0


def time_steps(step, flush, stream, steps, dev):
    """CUDA events on the launching stream around each step, L2 flushed between
    steps (outside the events); returns total ms."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    return sum(a.elapsed_time(b) for a, b in ev)


def compare_values(host_vals, host_status, dev_vals, dev_status, mode):
    """The host-entry results against the device path's.  Statuses must be
    equal; PARITY values bit-identical; SCORE values within the 1e-9 relative
    contract: on float capacities the large-graph builder's
    arc order — and with it the last bits of a push-relabel sum — can depend
    on warp scheduling."""
    import numpy as np
    hv_ = host_vals.numpy() if hasattr(host_vals, "numpy") else np.asarray(host_vals)
    dv_ = dev_vals.cpu().numpy()
    assert np.array_equal(np.asarray(host_status.numpy() if hasattr(host_status, "numpy") else host_status),
                          np.asarray(dev_status)), "e2e statuses differ"
    same = hv_.view(np.int64) == dv_.view(np.int64)
    rel = float(np.max(np.abs(hv_ - dv_) / np.maximum(1.0, np.abs(dv_)))) if hv_.size else 0.0
    assert rel <= (0.0 if mode == "parity" else 1e-9), f"e2e values differ (max rel {rel:.3g})"
    return {"bit_identical": int(same.sum()), "of": int(same.size), "max_rel_diff": rel}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="het42-70b")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: --global-batch split over the ranks (BASELINE configs[2]); "
                         "weak: --per-gpu candidates on every rank")
    ap.add_argument("--global-batch", type=int, default=None)
    ap.add_argument("--per-gpu", type=int, default=1_000_000)
    ap.add_argument("--ppm", type=int, default=0, help="uniform-interval mix, parts per million")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-routing", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--route-requests", type=int, default=1_000_000)
    ap.add_argument("--mode", default="score", choices=["score", "parity"],
                    help="headline scoring mode (the other mode is timed too and reported beside it)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.global_batch is None:
        args.global_batch = DEFAULT_BATCH.get(args.config, 100_000)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_01566_b200 as h
    from paper_2406_01566_b200 import clusters

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    # the JSON line is this process's only stdout: library chatter (NCCL's
    # version banner at communicator init) goes to stderr
    json_out = sys.stdout
    if world > 1:
        sys.stdout.flush()
        json_out = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    d = clusters.CONFIGS[args.config]("float")
    walk = args.config in WALK_CONFIGS
    headline = args.config == "het42-70b"
    c = h.Cluster.from_json(json.dumps(d))
    eng = h.Engine(c, device=local)
    eng.mode = args.mode
    N, L = eng.num_nodes, eng.num_layers
    first, B, G = shard(args, world, rank)
    # a dedicated stream: its handle is what the engine launches on, and the
    # CUDA events below are recorded on the same stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream

    def make_rows(first_, n_):
        t = torch.empty((n_, N, 2), dtype=torch.int16, device=dev)
        if walk:
            eng.generate_walk_device(SEED, first_, n_, t.data_ptr(), sp)
        else:
            eng.generate_device(SEED, first_, n_, args.ppm, t.data_ptr(), sp)
        return t

    pl = make_rows(first, B)
    vals = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    # the argmax writes its 16-byte record (value bits, global index) straight
    # into the all-gather's send buffer
    rec = torch.empty(2, dtype=torch.int64, device=dev)
    best = rec[0:1].view(torch.float64)
    bidx = rec[1:2]
    gathered = torch.empty(2 * world, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def step_on(rows, n, base, v, s):
        eng.score_device(rows.data_ptr(), n, v.data_ptr(), s.data_ptr(), True, sp)
        eng.argmax_device(v.data_ptr(), s.data_ptr(), n, base, best.data_ptr(), bidx.data_ptr(), sp)
        if world > 1:
            dist.all_gather_into_tensor(gathered, rec)

    def step():
        step_on(pl, B, first, vals, st)

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
    value = G / (ms_per_step / 1e3)  # every candidate of the global batch, over the slowest rank's time
    recs = unpack = None
    from paper_2406_01566_b200.dist import reduce_best, unpack_records
    recs = unpack_records(gathered) if world > 1 else [(float(best.item()), int(bidx.item()))]
    win = reduce_best(recs)
    st_host = st.cpu().numpy()
    head_vals = vals.clone()
    nonzero = float((head_vals > 0).double().mean().item())

    # the other mode on (a bounded prefix of) the same rows, same timing rules
    other = "parity" if args.mode == "score" else "score"
    ob = min(B, 1_000_000 if headline else 100_000)
    osteps = min(args.steps, 5)
    eng.mode = other
    ov = torch.empty(ob, dtype=torch.float64, device=dev)
    os_ = torch.empty(ob, dtype=torch.int32, device=dev)
    ostep = lambda: step_on(pl, ob, first, ov, os_)  # noqa: E731
    ostep()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ot = torch.tensor([time_steps(ostep, flush, stream, osteps, dev)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ot, op=dist.ReduceOp.MAX)
    other_rate = (ob * world) / (float(ot.item()) / osteps / 1e3)
    eng.mode = args.mode
    hv_ = head_vals[:ob]
    rel = ((hv_ - ov).abs() / ov.abs().clamp(min=1.0)).max().item() if ob else 0.0

    # weak scaling beside the strong headline: --per-gpu candidates on every rank
    weak = None
    if args.scaling == "strong" and world > 1 and not args.no_weak:
        wB = args.per_gpu
        wpl = make_rows(rank * wB, wB)
        wv = torch.empty(wB, dtype=torch.float64, device=dev)
        ws = torch.empty(wB, dtype=torch.int32, device=dev)
        wstep = lambda: step_on(wpl, wB, rank * wB, wv, ws)  # noqa: E731
        for _ in range(2):
            wstep()
        torch.cuda.synchronize(dev)
        dist.barrier()
        wt = torch.tensor([time_steps(wstep, flush, stream, args.steps, dev)], dtype=torch.float64, device=dev)
        dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        wms = float(wt.item()) / args.steps
        weak = {"value": wB * world / (wms / 1e3), "unit": "evals/s", "candidates_per_gpu": wB,
                "global_batch": wB * world, "ms_per_step": wms}
        del wpl, wv, ws

    # the winner's plan reaches every rank: its owner
    # computes the PARITY per-edge flows and broadcasts row + flows over NCCL
    winner_plan = None
    if world > 1 and win[1] >= 0:
        from paper_2406_01566_b200.dist import owner_of, share_winner
        owner = owner_of(win[1], [shard(args, world, r)[0] for r in range(world)])
        row_w = flows_w = None
        if owner == rank:
            row_w = pl[win[1] - first].cpu().numpy()
            _, _, _, ne_w, _, dbl_w = eng.flows(row_w[None], True)
            flows_w = dbl_w[0, :int(ne_w[0]), 1]
        t_share = time.perf_counter()
        row_s, flows_s = share_winner(owner, row_w, flows_w, N)
        winner_plan = {"owner_rank": owner, "edges": int(flows_s.size),
                       "bytes": int(row_s.nbytes + flows_s.nbytes),
                       "ms": (time.perf_counter() - t_share) * 1e3}

    # e2e through the C ABI with host buffers, timed on the host: the same rows
    # copied to pinned host memory (and to pageable memory for the second leg)
    e2e = e2e_pageable = None
    if not args.no_e2e:
        host = torch.empty((B, N, 2), dtype=torch.int16, pin_memory=True)
        host.copy_(pl)
        hv = torch.empty(B, dtype=torch.float64, pin_memory=True)
        hs = torch.empty(B, dtype=torch.int32, pin_memory=True)

        def e2e_time(hin, hval, hst, steps):
            for _ in range(2):
                eng.score_best_host_ptr(hin.data_ptr(), B, hval.data_ptr(), hst.data_ptr(), True)
            times, res = [], None
            for _ in range(steps):
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                res = eng.score_best_host_ptr(hin.data_ptr(), B, hval.data_ptr(), hst.data_ptr(), True)
                times.append(time.perf_counter() - t0)
            tt = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return G * steps / float(tt.item()), res

        e2e_rate, e2e_best = e2e_time(host, hv, hs, args.steps)
        check = compare_values(hv, hs, head_vals, st_host, args.mode)
        if world == 1:
            assert int(e2e_best[1]) == win[1] or abs(float(e2e_best[0]) - win[0]) <= 1e-9 * abs(win[0]), \
                "e2e winner differs from the device path"
        e2e = {"value": e2e_rate, "unit": "evals/s", "h2d_bytes_per_step": G * 4 * N,
               "d2h_bytes_per_step": G * 12 + 16 * world,
               "call": "helio_gpu_score_best_host (pinned host placements in; every value + status and the "
                       "first-max winner out)", "check_vs_device": check}
        # pageable buffers (what Engine.score and a plain ctypes caller pass):
        # the entry stages chunks through its own pinned buffers
        hp = torch.empty((B, N, 2), dtype=torch.int16)
        hp.copy_(host)
        del host
        hvp = torch.empty(B, dtype=torch.float64)
        hsp = torch.empty(B, dtype=torch.int32)
        prate, _ = e2e_time(hp, hvp, hsp, min(args.steps, 5))
        pcheck = compare_values(hvp, hsp, head_vals, st_host, args.mode)
        e2e_pageable = {"value": prate, "unit": "evals/s", "h2d_bytes_per_step": G * 4 * N,
                        "d2h_bytes_per_step": G * 12 + 16 * world,
                        "call": "helio_gpu_score_best_host with pageable host buffers (staged)",
                        "check_vs_device": pcheck}
        del hp, hvp, hsp

    # extras (single-GPU views of the headline cluster) only at N = 1: at N > 1
    # the other ranks must not wait on rank 0 outside the timed region
    extras = world == 1 and headline and not args.no_configs
    split = cfg_table = routing = search = None
    if extras:
        for name, fn in (("split", lambda: split_leg(eng, local, sp)),
                         ("cfg", lambda: config_table(h, clusters, local, sp, with_reference=not args.no_cpu_baseline)),
                         ("search", lambda: search_leg(h, clusters, local))):
            try:
                r = fn()
            except Exception as ex:  # reported, never fatal
                r = {"error": str(ex)}
            if name == "split":
                split = r
            elif name == "cfg":
                cfg_table = r
            else:
                search = r
    latency = None
    if extras:
        try:
            latency = latency_leg(h, clusters, with_reference=not args.no_cpu_baseline)
        except Exception as ex:  # reported, never fatal
            latency = {"error": str(ex)}
    if world == 1 and headline and not args.no_routing:
        try:
            routing = routing_leg(h, clusters, local, sp, args.route_requests, with_reference=not args.no_cpu_baseline)
        except Exception as ex:  # reported, never fatal
            routing = {"value": None, "error": str(ex)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_baseline(d, walk, args.cpu_seconds, args.ppm)
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

    # roofline of the dominant kernel (fused build + solve).  The binding
    # resource is warp-instruction issue: warp-instructions per
    # candidate from the committed ncu capture x candidates per launch / the
    # live kernel time, against SMs x 4 schedulers x the sampled SM clock.
    # HBM (SURVEY §8(d) fused formula 4N + 8, + 4 B status) is kept beside it.
    bytes_per_eval = 4 * N + 8 + 4
    kms = [k for k in kernel_ms if k and k > 0]
    avg_kernel_ms = sum(kms) / len(kms) if kms else ms_per_step
    hbm_ach = bytes_per_eval * B / (avg_kernel_ms / 1e3) / 1e9
    peak, peak_src = load_peaks()
    tpe, tsrc, tgraphs = ncu_traffic_per_eval(args.config, args.mode)
    ipe = ncu_inst_per_eval(args.config, args.mode)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clocks.get("sm_mhz") or 1965.0
    issue_peak = sms * 4 * mhz * 1e6
    issue_ach = ipe * B / (avg_kernel_ms / 1e3) if ipe else None
    roofline = {"bound": "issue", "achieved": issue_ach, "peak": issue_peak, "unit": "warp-instr/s",
                "frac": (issue_ach / issue_peak) if issue_ach else None,
                "issue_frac": (issue_ach / issue_peak) if issue_ach else None,
                "warp_instr_per_eval": ipe,
                "issue_source": "smsp__inst_executed.sum per candidate from the committed ncu capture; peak = SMs x "
                                "4 schedulers x median SM clock under load",
                "traffic": (tpe * B) if tpe is not None else None,
                "traffic_unit": "bytes per launch (DRAM read + write)",
                "traffic_source": (f"{tsrc}: ncu --set full of one {tgraphs}-candidate launch, per candidate x {B}"
                                   if tsrc else "no committed capture for this config/mode"),
                "hbm_achieved": hbm_ach, "hbm_peak": peak, "hbm_unit": "GB/s", "hbm_frac": hbm_ach / peak,
                "hbm_peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_per_eval * B,
                "bytes_per_eval": bytes_per_eval,
                "kernel": f"score_kernel<{args.mode}> (fused K1 build + K2 solve; small/middle/big slot tiers)",
                "kernel_ms": avg_kernel_ms, "kernel_share_of_step": avg_kernel_ms / ms_per_step}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, world),
            "details": {"mode": args.mode,
                        "other_mode": {"mode": other, "value": other_rate, "unit": "evals/s", "candidates": ob,
                                       "max_rel_diff_vs_headline": rel},
                        "nonzero_fraction": nonzero, "status_nonzero": int((st_host != 0).sum()),
                        "best": {"value": win[0], "index": win[1]}, "winner_plan_broadcast": winner_plan,
                        "inputs_bytes_per_gpu": B * 4 * N},
            "weak_scaling": weak,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable,
            "gpu_launches": launches,
            "routing": routing, "latency": latency, "other_configs": cfg_table, "split_pipeline": split,
            "search": search,
            "clocks": clocks,
        }
        print(json.dumps(out), file=json_out, flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
