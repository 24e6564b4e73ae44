"""Test-only helpers: golden-file loader, CSR from edge lists, brute-force checkers.

The brute-force checkers are independent of oracle/oracle.c (pure Python / numpy,
structurally different algorithms: path enumeration, memoised DFS, vectorised
fix-point relaxation) so they can pin the oracle.
"""
from __future__ import annotations

import os
import sys

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
F32 = np.float32


def load_golden(name):
    out = {"edge": []}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, *vals = line.split()
            vals = [int(v) for v in vals]
            if k == "edge":
                out["edge"].append(tuple(vals))
            else:
                out[k] = vals if len(vals) != 1 else vals[0]
    return out


def csr_from_edges(n, edges):
    """Fan-in CSR (rows = sink) keeping edge-list order within a row."""
    edges = list(edges)
    dst = np.array([v for _, v in edges], dtype=np.int64)
    src = np.array([u for u, _ in edges], dtype=np.int64)
    order = np.argsort(dst, kind="stable") if len(edges) else np.zeros(0, np.int64)
    counts = np.bincount(dst, minlength=n) if len(edges) else np.zeros(n, np.int64)
    in_ptr = np.zeros(n + 1, np.int32)
    in_ptr[1:] = np.cumsum(counts)
    return in_ptr, src[order].astype(np.int32), order


def random_tiny_dag(rng, nmax=8, p=0.45, multi=0.15):
    """Random DAG from a hidden topological order, random relabel, optional multi-edges."""
    n = int(rng.integers(1, nmax + 1))
    topo = rng.permutation(n)
    edges = []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < p:
                edges.append((int(topo[i]), int(topo[j])))
                if rng.random() < multi:
                    edges.append((int(topo[i]), int(topo[j])))
    rng.shuffle(edges)
    return n, edges


def mixed_delays(rng, m):
    mag = 10.0 ** rng.uniform(-3, 3, size=m)
    sign = np.where(rng.random(m) < 0.3, -1.0, 1.0)
    return (mag * sign).astype(np.float32)


def brute_paths(n, edges_with_delay):
    """All source->v paths as lists of edge indices (tiny graphs only)."""
    ins = [[] for _ in range(n)]
    for k, (u, v, _) in enumerate(edges_with_delay):
        ins[v].append(k)
    sys.setrecursionlimit(10000)
    memo = {}

    def paths_to(v):
        if v in memo:
            return memo[v]
        if not ins[v]:
            res = [[]]
        else:
            res = []
            for k in ins[v]:
                u = edges_with_delay[k][0]
                for p in paths_to(u):
                    res.append(p + [k])
        memo[v] = res
        return res

    return [paths_to(v) for v in range(n)]


def brute_forward(n, edges_with_delay, at_src, early=False):
    """at[v] = max (early: min) over source->v paths of the left-to-right fp32 path
    sum (P6, P12)."""
    allp = brute_paths(n, edges_with_delay)
    at = np.zeros(n, F32)
    level = np.zeros(n, np.int64)
    for v in range(n):
        best = None
        for p in allp[v]:
            start = edges_with_delay[p[0]][0] if p else v
            x = F32(at_src[start])
            if x == 0:
                x = F32(0.0)
            for k in p:
                x = F32(x + F32(edges_with_delay[k][2]))
            if best is None or (x < best if early else x > best):
                best = x
        at[v] = best
        level[v] = max(len(p) for p in allp[v])
    return at, level


def brute_backward(n, edges_with_delay, T, early=False):
    """rat[u] = min (early: max) over u->sink paths of fp32 differences applied from
    the sink (P6, P12)."""
    outs = [[] for _ in range(n)]
    for k, (u, v, _) in enumerate(edges_with_delay):
        outs[u].append(k)
    memo = {}

    def paths_from(u):
        if u in memo:
            return memo[u]
        if not outs[u]:
            res = [[]]
        else:
            res = []
            for k in outs[u]:
                for p in paths_from(edges_with_delay[k][1]):
                    res.append([k] + p)
        memo[u] = res
        return res

    rat = np.zeros(n, F32)
    for u in range(n):
        best = None
        for p in paths_from(u):
            x = F32(T)
            for k in reversed(p):
                x = F32(x - F32(edges_with_delay[k][2]))
            if best is None or (x > best if early else x < best):
                best = x
        rat[u] = best
    return rat


def fixpoint_levels(n, src, dst):
    """level[v] = longest path (edges) from a source by vectorised Bellman-Ford
    fix-point (numpy, not Kahn); None if it does not converge within n+1 rounds."""
    lv = np.zeros(n, np.int64)
    for _ in range(n + 1):
        cand = np.zeros(n, np.int64)
        if len(src):
            np.maximum.at(cand, dst, lv[src] + 1)
        new = np.maximum(lv, cand)
        if np.array_equal(new, lv):
            return lv
        lv = new
    return None


def fixpoint_heights(n, src, dst):
    """height[u] = longest path (edges) from u to a sink."""
    return fixpoint_levels(n, dst, src)


def dfs_int_at(n, src, dst, d_int, at_src_int):
    """Exact integer longest-path arrival by memoised DFS over fan-in (P8)."""
    ins = [[] for _ in range(n)]
    for e in range(len(src)):
        ins[dst[e]].append(e)
    memo = [None] * n
    for root in range(n):
        stack = [(root, False)]
        while stack:
            v, expanded = stack.pop()
            if memo[v] is not None:
                continue
            if not ins[v]:
                memo[v] = int(at_src_int[v])
                continue
            if expanded:
                memo[v] = max(memo[src[e]] + int(d_int[e]) for e in ins[v])
            else:
                stack.append((v, True))
                for e in ins[v]:
                    if memo[src[e]] is None:
                        stack.append((int(src[e]), False))
    return memo


def dfs_int_rat(n, src, dst, d_int, T):
    outs = [[] for _ in range(n)]
    for e in range(len(src)):
        outs[src[e]].append(e)
    memo = [None] * n
    for root in range(n):
        stack = [(root, False)]
        while stack:
            u, expanded = stack.pop()
            if memo[u] is not None:
                continue
            if not outs[u]:
                memo[u] = int(T)
                continue
            if expanded:
                memo[u] = min(memo[dst[e]] - int(d_int[e]) for e in outs[u])
            else:
                stack.append((u, True))
                for e in outs[u]:
                    if memo[dst[e]] is None:
                        stack.append((int(dst[e]), False))
    return memo


def reach_from_cycles(n, edges):
    """Nodes reachable from (or on) a directed cycle: exactly the nodes Kahn never
    makes ready.  Brute force via transitive closure (tiny graphs)."""
    R = np.zeros((n, n), bool)
    for u, v in edges:
        R[u, v] = True
    for k in range(n):
        R |= R[:, k:k + 1] & R[k:k + 1, :]
    on_cycle = np.diag(R).copy()
    bad = on_cycle.copy()
    for c in np.nonzero(on_cycle)[0]:
        bad |= R[c]
    return bad
