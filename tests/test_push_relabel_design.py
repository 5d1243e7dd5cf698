"""CPU check of the SCORE push-relabel design (solve_score.cuh solve_pr +
pr_global_relabel) against the oracle.

The kernel's algorithm — preflow phase only, FIFO batches of up to 32 live
vertices, one admissible push per lane per round with the lowest lane winning
a shared target, sink deposits summed at the end, relabel to 1 + min residual
neighbour height capped at n, early-stopping backward-BFS global relabels that
give the unlabelled rest (head level + 1) — is restated here step for step in
plain Python and run on the reference's own graphs (oracle build of syn256 link
walks and AC1 raw graphs).  The value must equal the reference's max-flow (exact
on integer capacities, 1e-9 relative on float), which pins the design choices
that the GPU parity tests then pin for the kernel itself.
"""

from __future__ import annotations

import os
import sys
from collections import deque


sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))

from _support import Oracle, golden, max_flow_raw_oracle  # noqa: E402

EPS = 1e-12  # FLOW_EPS, flow_graph.cpp:15


def _residual(n, us, vs, caps):
    """Arcs as the SCORE builder lays them out (forward at u, reverse at v)."""
    adj = [[] for _ in range(n)]
    to, cap, rev = [], [], []
    for u, v, c in zip(us, vs, caps):
        a = len(to)
        to += [int(v), int(u)]
        cap += [float(c), 0.0]
        rev += [a + 1, a]
        adj[int(u)].append(a)
        adj[int(v)].append(a + 1)
    return adj, to, cap, rev


def _global_relabel(n, s, t, adj, to, cap, rev, h, ex):
    need = 0
    for x in range(n):
        dead = x == s or h[x] >= n
        if not dead and x != t and ex[x] > 0.0:
            need += 1
        h[x] = n if dead else -1
    h[t] = 0
    q = [t]
    qh, off = 0, 0  # queue head and arcs of q[qh] already scanned
    while qh < len(q):
        # one warp step: the next 32 arcs of the queue's arc stream
        arcs, k, o = [], qh, off
        while k < len(q) and len(arcs) < 32:
            lst = adj[q[k]][o:]
            room = 32 - len(arcs)
            if len(lst) <= room:
                arcs += [(q[k], a) for a in lst]
                k, o = k + 1, 0
            else:
                arcs += [(q[k], a) for a in lst[:room]]
                o += room
        seen = set()
        for v, a in arcs:  # lanes in stream order; the lowest lane wins a duplicate
            x = to[a]
            if h[x] == -1 and cap[rev[a]] > EPS and x not in seen:
                seen.add(x)
                h[x] = h[v] + 1
                q.append(x)
                if ex[x] > 0.0:
                    need -= 1
        qh, off = k, o
        if need == 0 and qh < len(q):
            break
    rest = h[q[qh]] + 1 if qh < len(q) else n
    for x in range(n):
        if h[x] == -1:
            h[x] = rest


def push_relabel_value(n, s, t, us, vs, caps, gr_every=20):
    adj, to, cap, rev = _residual(n, us, vs, caps)
    ex = [0.0] * n
    h = [0] * n
    inq = [False] * n
    fifo = deque()
    for a in adj[s]:  # saturate the source's arcs in adjacency order
        c = cap[a]
        if c > 0.0:
            v = to[a]
            cap[a] = 0.0
            cap[rev[a]] += c
            ex[v] += c
            if v not in (s, t) and not inq[v]:
                inq[v] = True
                fifo.append(v)
    sink = [0.0] * 32
    since = gr_every
    while fifo:
        if since >= gr_every:
            _global_relabel(n, s, t, adj, to, cap, rev, h, ex)
            since = 0
        since += 1
        lanes = []
        for lane in range(min(32, len(fifo))):
            u = fifo.popleft()
            inq[u] = False
            if h[u] < n and ex[u] > 0.0:
                lanes.append([lane, u, 0, h[u]])
        while True:
            want = []
            for L in lanes:
                lane, u, i, hu = L
                if ex[u] <= 0.0:
                    continue
                al = adj[u]
                while i < len(al) and not (h[to[al[i]]] == hu - 1 and cap[al[i]] > EPS):
                    i += 1
                L[2] = i
                if i < len(al):
                    want.append(L)
            if not want:
                break
            taken, deposits = set(), []
            for L in want:  # lane order; lowest lane per non-sink target
                lane, u, i, hu = L
                a = adj[u][i]
                v = to[a]
                if v != t and v in taken:
                    continue
                taken.add(v)
                e, c = ex[u], cap[a]
                d = c if c < e else e
                cap[a] = c - d
                cap[rev[a]] += d
                ex[u] = e - d
                if v == t:
                    sink[lane] += d
                else:
                    deposits.append(v)
                    deposits.append(d)
                if d == c:
                    L[2] = i + 1
            for j in range(0, len(deposits), 2):
                v, d = deposits[j], deposits[j + 1]
                ex[v] += d
                if not inq[v]:
                    inq[v] = True
                    fifo.append(v)
        new = {}
        for lane, u, i, hu in lanes:
            if ex[u] > 0.0:
                best = n
                for a in adj[u]:
                    if cap[a] > EPS:
                        best = min(best, h[to[a]] + 1)
                new[u] = best
        for u, b in new.items():
            h[u] = b
            if b < n and not inq[u]:
                inq[u] = True
                fifo.append(u)
    # the kernel's shuffle-xor tree over the 32 lane sums
    vals = list(sink)
    for o in (16, 8, 4, 2, 1):
        vals = [vals[i] + vals[i ^ o] for i in range(32)]
    return ex[t] + vals[0]


def _check(val, ref, integer):
    if integer:
        assert val == ref, (val, ref)
    else:
        assert abs(val - ref) <= 1e-9 * max(1.0, abs(ref)), (val, ref)


def test_design_on_syn256_link_walks():
    from make_golden import walk_rows
    from paper_2406_01566_b200 import clusters

    for cap in ("float", "int"):
        d = clusters.CONFIGS["syn256-120l"](cap)
        o = Oracle(d)
        rows = walk_rows(d, o.kmax(), 11, 3)
        nonzero = 0
        for r in rows:
            st, nv, E, val = o.graph(r, True)
            assert st == 0
            got = push_relabel_value(nv, 0, 1, E["u"], E["v"], E["cap"])
            _check(got, val, cap == "int")
            nonzero += val > 0
        assert nonzero >= 2


def test_design_on_raw_graphs():
    g = golden("raw_ac1.npz")
    for i in range(0, 200, 7):
        n, s, t = int(g["n"][i]), int(g["s"][i]), int(g["t"][i])
        a, b = int(g["off"][i]), int(g["off"][i + 1])
        u, v, c = g["u"][a:b], g["v"][a:b], g["cap"][a:b]
        ref, _ = max_flow_raw_oracle(n, s, t, u, v, c)
        got = push_relabel_value(n, s, t, u, v, c, gr_every=3)
        assert abs(got - ref) <= 1e-9 * max(1.0, abs(ref)), (i, got, ref)
