"""Pins for the CPU oracle.  CPU only.

Each test ties oracle/ to something other than itself: the paper's worked graphs
(tests/golden/, cited), closed forms, generator-known levels, brute-force path
enumeration, exact integer DFS, invariants and metamorphic relations.
"""
import itertools

import numpy as np
import pytest

import hfgen
import oracle
from helpers import (brute_backward, brute_forward, csr_from_edges, dfs_int_at,
                     dfs_int_rat, fixpoint_heights, fixpoint_levels, load_golden,
                     mixed_delays, random_tiny_dag, reach_from_cycles)

F32 = np.float32


# ---- P1: Fig. 1 / Listing 1 saxpy graph ------------------
def test_p1_fig1_levels_and_order():
    g = load_golden("fig1_saxpy.txt")
    in_ptr, in_src, _ = csr_from_edges(g["n"], g["edge"])
    assert len(g["edge"]) == 6
    lv = oracle.levelize(g["n"], len(g["edge"]), in_ptr, in_src)
    assert lv.level.tolist() == g["level"]
    assert lv.num_levels == g["num_levels"]
    assert lv.level_ptr.tolist() == g["level_ptr"]
    assert lv.order.tolist() == g["order"]


def _run_saxpy(schedule, N, x0, y0, a):
    """Execute Listing 1's seven payloads in `schedule` order."""
    st = {}
    payload = {
        0: lambda: st.__setitem__("x", np.full(N, x0, np.int64)),          # host_x
        1: lambda: st.__setitem__("y", np.full(N, y0, np.int64)),          # host_y
        2: lambda: st.__setitem__("dx", st["x"].copy()),                    # pull_x
        3: lambda: st.__setitem__("dy", st["y"].copy()),                    # pull_y
        4: lambda: st.__setitem__("dy", a * st["dx"] + st["dy"]),           # kernel saxpy
        5: lambda: st.__setitem__("x", st["dx"].copy()),                    # push_x
        6: lambda: st.__setitem__("y", st["dy"].copy()),                    # push_y
    }
    for t in schedule:
        payload[int(t)]()
    return st["y"]


def test_p1_fig1_saxpy_result_in_canonical_order():
    g = load_golden("fig1_saxpy.txt")
    in_ptr, in_src, _ = csr_from_edges(g["n"], g["edge"])
    lv = oracle.levelize(g["n"], len(g["edge"]), in_ptr, in_src)
    y = _run_saxpy(lv.order, g["N"], g["x"], g["y"], g["a"])
    assert np.all(y == g["result_y"])          # y = 2*1 + 2 = 4 (BASELINE.json:5)
    y_fifo = _run_saxpy(lv.topo, g["N"], g["x"], g["y"], g["a"])
    assert np.all(y_fifo == g["result_y"])
    # negative control: push_y before the kernel observes y = 2
    bad = [0, 1, 2, 3, 6, 4, 5]
    assert np.all(_run_saxpy(bad, g["N"], g["x"], g["y"], g["a"]) == 2)


# ---- P2: Fig. 5 / Listing 10 ----------------------------
def test_p2_fig5_levels_and_transitive_edge():
    g = load_golden("fig5_dependency.txt")
    assert g["n"] == 8 and len(g["edge"]) == 7      # "eight tasks and seven constraints"
    in_ptr, in_src, _ = csr_from_edges(g["n"], g["edge"])
    lv = oracle.levelize(g["n"], 7, in_ptr, in_src)
    assert lv.level.tolist() == g["level"]
    assert lv.level_ptr.tolist() == g["level_ptr"]
    assert lv.order.tolist() == g["order"]
    # without kernel1->kernel2, kernel2 (7) no longer follows kernel1 (6)
    edges = [e for e in g["edge"] if e != (6, 7)]
    ip, isrc, _ = csr_from_edges(8, edges)
    lv2 = oracle.levelize(8, 6, ip, isrc)
    assert lv2.level[7] == lv2.level[6] == 2


# ---- P3: unit-delay identity ----------------------------------------------
@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C2-random", 0.01), ("C3", 0.01)])
def test_p3_unit_delay_identity(name, scale):
    g = hfgen.config(name, scale)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    ones = np.ones(g.m, F32)
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, ones, np.zeros(g.n, F32), lv)
    assert np.array_equal(at, lv.level.astype(F32))
    src, dst = g.edges()
    height = fixpoint_heights(g.n, src, dst)
    T = float(lv.num_levels - 1)
    rat, slack, wns = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, ones, T, at, lv)
    assert np.array_equal(rat, (lv.num_levels - 1 - height).astype(F32))
    assert wns == F32(0.0) and np.all(slack >= 0)


# ---- P4: closed forms ------------------------------------------------------
def test_p4_chain_closed_form():
    g = hfgen.chain(5000, seed=2, relabel=True)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    assert lv.num_levels == 5000
    # recover positions: walk from the unique source
    src, dst = g.edges()
    nxt = np.full(g.n, -1, np.int64)
    nxt[src] = dst
    head = int(np.setdiff1d(np.arange(g.n), dst)[0])
    pos = np.empty(g.n, np.int64)
    v = head
    for k in range(g.n):
        pos[v] = k
        v = nxt[v]
    assert np.array_equal(lv.level, pos)
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, np.ones(g.m, F32), None, lv)
    assert np.array_equal(at, pos.astype(F32))            # exact below 2^24
    assert np.array_equal(lv.order, np.argsort(pos))      # one node per level


def test_p4_bintree_closed_form():
    n = 1_000_000
    g = hfgen.bintree(n, seed=2, relabel=False)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    expect = np.array([int(i + 1).bit_length() - 1 for i in range(0, n, 997)])
    assert np.array_equal(lv.level[::997], expect)
    assert lv.num_levels == 20
    # in-tree (reversed edges): leaves are sources
    src, dst = g.edges()
    ip, isrc, _ = csr_from_edges(n, list(zip(dst.tolist(), src.tolist())))
    lv2 = oracle.levelize(n, g.m, ip, isrc)
    assert lv2.level[0] == 19


# ---- P5: generator-known levels --------------------------------------------
@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C3", 0.05), ("C3", 1.0)])
def test_p5_generator_levels(name, scale):
    g = hfgen.config(name, scale)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    assert np.array_equal(lv.level, g.level_label)
    assert lv.num_levels == g.depth


# ---- P6: brute force on tiny DAGs -----------------------------------------
def test_p6_bruteforce_tiny_dags():
    rng = np.random.default_rng(2203)
    for trial in range(1500):
        n, edges = random_tiny_dag(rng)
        m = len(edges)
        d = mixed_delays(rng, m)
        at_src = mixed_delays(rng, n)
        T = float(mixed_delays(rng, 1)[0])
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        d_csr = d[perm]
        ewd = [(u, v, d[k]) for k, (u, v) in enumerate(edges)]
        at_b, lev_b = brute_forward(n, ewd, at_src)
        rat_b = brute_backward(n, ewd, T)
        lv = oracle.levelize(n, m, in_ptr, in_src)
        assert np.array_equal(lv.level, lev_b), trial
        at = oracle.forward(n, m, in_ptr, in_src, d_csr, at_src, lv)
        assert np.array_equal(at.view(np.uint32), at_b.view(np.uint32)), trial
        rat, slack, wns = oracle.backward(n, m, in_ptr, in_src, d_csr, T, at, lv)
        assert np.array_equal(rat.view(np.uint32), rat_b.view(np.uint32)), trial
        s_b = (rat_b - at_b).astype(F32)
        assert np.array_equal(slack.view(np.uint32), s_b.view(np.uint32))
        assert wns == s_b.min()


def test_p6_cycles_count_unready_nodes():
    rng = np.random.default_rng(7)
    found = 0
    for trial in range(400):
        n, edges = random_tiny_dag(rng, nmax=8)
        if n < 2:
            continue
        # inject back edges / self loops
        for _ in range(int(rng.integers(1, 3))):
            u = int(rng.integers(0, n))
            v = int(rng.integers(0, n))
            edges.append((u, v))
        bad = reach_from_cycles(n, edges)
        in_ptr, in_src, _ = csr_from_edges(n, edges)
        if bad.any():
            found += 1
            with pytest.raises(oracle.OracleError) as ei:
                oracle.levelize(n, len(edges), in_ptr, in_src)
            assert ei.value.code == oracle.CYCLE
            assert ei.value.unready == int(bad.sum())
        else:
            oracle.levelize(n, len(edges), in_ptr, in_src)
    assert found > 100


# ---- P7: invariants ---------------------------------------------------------
@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C2-random", 0.02), ("C5", 0.002)])
def test_p7_invariants(name, scale):
    g = hfgen.config(name, scale)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    src, dst = g.edges()
    L = lv.level
    assert np.all(L[src] < L[dst])
    best = np.full(g.n, -1, np.int64)
    np.maximum.at(best, dst, L[src])
    assert np.array_equal(L, best + 1)                   # level = 1 + max pred level
    sizes = np.diff(lv.level_ptr)
    assert np.all(sizes > 0) and sizes.sum() == g.n
    for k in range(lv.num_levels):                      # ascending ids within level
        seg = lv.order[lv.level_ptr[k]:lv.level_ptr[k + 1]]
        assert np.all(np.diff(seg) > 0) and np.all(L[seg] == k)
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
    x = (at[src] + g.delay).astype(F32)
    assert np.all(at[dst] >= x)
    tight = np.zeros(g.n, bool)
    tight[dst[at[dst] == x]] = True
    indeg = np.diff(g.in_ptr)
    assert np.all(tight[indeg > 0])
    rat, slack, wns = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, at, lv)
    y = (rat[dst] - g.delay).astype(F32)
    assert np.all(rat[src] <= y)
    tight = np.zeros(g.n, bool)
    tight[src[rat[src] == y]] = True
    outdeg = np.bincount(src, minlength=g.n)
    assert np.all(tight[outdeg > 0])
    assert np.all(rat[outdeg == 0] == F32(g.t_req))
    assert wns == slack.min() and np.array_equal(slack, (rat - at).astype(F32))


def test_p7_fixpoint_levels_agree():
    g = hfgen.config("C2-random", 0.01)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    src, dst = g.edges()
    assert np.array_equal(lv.level, fixpoint_levels(g.n, src, dst))


# ---- P8: exact-integer sums vs memoised DFS ---------------------------------
@pytest.mark.parametrize("name,scale", [("C1", 0.3), ("C5", 0.0005)])
def test_p8_exact_integer_dfs(name, scale):
    g = hfgen.config(name, scale)
    rng = np.random.default_rng(8)
    d_int = rng.integers(1, 65, size=g.m)
    a_int = rng.integers(0, 100, size=g.n)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, d_int.astype(F32), a_int.astype(F32), lv)
    src, dst = g.edges()
    exp = dfs_int_at(g.n, src.tolist(), dst.tolist(), d_int.tolist(), a_int.tolist())
    assert np.array_equal(at, np.array(exp, dtype=F32))
    T = 100000
    rat, _, _ = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, d_int.astype(F32), T, at, lv)
    expr = dfs_int_rat(g.n, src.tolist(), dst.tolist(), d_int.tolist(), T)
    assert np.array_equal(rat, np.array(expr, dtype=F32))


# ---- P9: metamorphic ---------------------------------------------------------
def test_p9_monotone_and_batch_equals_single():
    g = hfgen.config("C1")
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
    rat, slack, wns = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, at, lv)
    rng = np.random.default_rng(9)
    for _ in range(5):
        d2 = g.delay.copy()
        e = int(rng.integers(0, g.m))
        d2[e] = F32(d2[e] * 3.0)
        at2 = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, d2, g.at_src, lv)
        assert np.all(at2 >= at)
    S = 6
    D = hfgen.scenario_delays(g, 0, S, "ms")
    D[:, 3] = g.delay                                   # scenario 3 = base delays
    T = np.full(S, g.t_req, F32)
    for layout, arr in (("ms", D), ("sm", np.ascontiguousarray(D.T))):
        w, at_all, rat_all = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, arr, T, g.at_src,
                                          layout=layout, threads=3, want_at_rat=True)
        assert np.array_equal(at_all[:, 3].view(np.uint32), at.view(np.uint32))
        assert np.array_equal(rat_all[:, 3].view(np.uint32), rat.view(np.uint32))
        assert w[3] == wns
        for s in range(S):
            a_s = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, D[:, s], g.at_src, lv)
            _, _, w_s = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, D[:, s], g.t_req, a_s, lv)
            assert w[s] == w_s
    w1 = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, threads=1)
    w4 = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, threads=4)
    assert np.array_equal(w1, w4)


# ---- P10: endpoint WNS sanity (tolerance, not the contract) -----------------
def test_p10_endpoint_wns():
    g = hfgen.config("C1")
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
    _, _, wns = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, at, lv)
    sinks = np.bincount(g.in_src, minlength=g.n) == 0
    approx = np.float64(g.t_req) - np.float64(at[sinks].max())
    assert abs(float(wns) - approx) <= 1e-5 * max(1.0, abs(approx)) + 64 * np.spacing(F32(g.t_req))


# ---- edge cases ----------------------------------------------------------------
def test_edge_cases_empty_and_isolated():
    lv = oracle.levelize(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32))
    assert lv.num_levels == 0 and lv.level_ptr.tolist() == [0]
    rat, slack, wns = oracle.backward(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32),
                                      None, 5.0, np.zeros(0, np.float32), lv)
    assert np.isinf(wns) and wns > 0
    # isolated nodes: sources and sinks at once
    ip = np.zeros(4, np.int32)
    lv = oracle.levelize(3, 0, ip, np.zeros(0, np.int32))
    at = oracle.forward(3, 0, ip, np.zeros(0, np.int32), None, np.array([1, -0.0, 3], F32), lv)
    assert at.view(np.uint32).tolist() == np.array([1, 0.0, 3], F32).view(np.uint32).tolist()
    rat, slack, wns = oracle.backward(3, 0, ip, np.zeros(0, np.int32), None, -0.0, at, lv)
    assert rat.view(np.uint32).tolist() == [0, 0, 0]
    assert wns == F32(-3.0)


def test_edge_cases_invalid_inputs():
    ip, isrc, _ = csr_from_edges(3, [(0, 1), (1, 2)])
    lv = oracle.levelize(3, 2, ip, isrc)
    with pytest.raises(oracle.OracleError):
        oracle.forward(3, 2, ip, isrc, np.array([1, np.nan], F32), None, lv)
    with pytest.raises(oracle.OracleError):
        oracle.forward(3, 2, ip, isrc, np.array([1, np.inf], F32), None, lv)
    assert oracle.check_csr(3, 2, np.array([0, 0, 1, 3], np.int32), isrc) == oracle.BAD_CSR
    assert oracle.check_csr(3, 2, ip, np.array([0, 3], np.int32)) == oracle.BAD_CSR
    assert oracle.check_csr(3, 2, np.array([0, 2, 1, 2], np.int32), isrc) == oracle.BAD_CSR


def test_fanout_check_multiset():
    g = hfgen.config("C1", 0.1)
    op, od, oe = oracle.fanout(g.n, g.m, g.in_ptr, g.in_src)
    src, dst = g.edges()
    assert np.array_equal(od, dst[oe]) and np.array_equal(g.in_src[oe], np.repeat(
        np.arange(g.n), np.diff(op)))
    assert np.all(np.diff(oe)[np.diff(np.repeat(np.arange(g.n), np.diff(op))) == 0] > 0)
    assert oracle.check_fanout(g.n, g.m, g.in_ptr, g.in_src, op, od) == oracle.OK
    od2 = od.copy()
    rng = np.random.default_rng(0)
    for u in range(g.n):                                   # shuffle inside rows: still OK
        rng.shuffle(od2[op[u]:op[u + 1]])
    assert oracle.check_fanout(g.n, g.m, g.in_ptr, g.in_src, op, od2) == oracle.OK
    k = int(np.nonzero(np.diff(op))[0][0])
    od3 = od.copy()
    od3[op[k]] = (od3[op[k]] + 1) % g.n
    assert oracle.check_fanout(g.n, g.m, g.in_ptr, g.in_src, op, od3) == oracle.BAD_CSR


# ---- P11: critical-path trace-back (NEXT-1, reading R17) --------------------------
def _greedy_int_path(n, src, dst, d_int, a_int, T):
    """Expected path in exact integer arithmetic: worst sink (T - at, ties by id), then
    the smallest fan-in edge id attaining the max, independently of the float code."""
    at = dfs_int_at(n, src, dst, d_int, a_int)
    outdeg = np.bincount(np.asarray(src, np.int64), minlength=n) if len(src) else np.zeros(n)
    sinks = [v for v in range(n) if outdeg[v] == 0]
    v = min(sinks, key=lambda u: (T - at[u], u))
    ins = [[] for _ in range(n)]
    for e in range(len(src)):
        ins[dst[e]].append(e)
    path = [v]
    while ins[v]:
        e = min(e for e in ins[v] if at[src[e]] + d_int[e] == at[v])
        v = src[e]
        path.append(v)
    return path


def test_p11_critical_path_integer_ties():
    # integer delays in [1, 4]: many exact ties, so the tie rules are exercised
    rng = np.random.default_rng(11)
    for trial in range(400):
        n, edges = random_tiny_dag(rng, nmax=10, p=0.5)
        m = len(edges)
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        dst = np.repeat(np.arange(n), np.diff(in_ptr)).astype(np.int64)
        d_int = rng.integers(1, 5, size=m)
        a_int = rng.integers(0, 3, size=n)
        T = 40
        at = oracle.forward(n, m, in_ptr, in_src, d_int.astype(F32), a_int.astype(F32))
        got = oracle.critical_path(n, m, in_ptr, in_src, d_int.astype(F32), at, T)
        exp = _greedy_int_path(n, in_src.tolist(), dst.tolist(), d_int.tolist(), a_int.tolist(), T)
        assert got.tolist() == exp, trial
    g = hfgen.config("C1", 0.3)
    d_int = rng.integers(1, 65, size=g.m)
    a_int = rng.integers(0, 100, size=g.n)
    src, dst = g.edges()
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, d_int.astype(F32), a_int.astype(F32))
    got = oracle.critical_path(g.n, g.m, g.in_ptr, g.in_src, d_int.astype(F32), at, 10 ** 6)
    exp = _greedy_int_path(g.n, src.tolist(), dst.tolist(), d_int.tolist(), a_int.tolist(), 10 ** 6)
    assert got.tolist() == exp


def test_p11_critical_path_bruteforce_fp32():
    # mixed-magnitude fp32 delays: the traced path is a real source -> worst-sink path
    # whose left-to-right fp32 sum is the brute-force maximum at the endpoint
    rng = np.random.default_rng(1102)
    for trial in range(400):
        n, edges = random_tiny_dag(rng)
        m = len(edges)
        d = mixed_delays(rng, m)
        at_src = mixed_delays(rng, n)
        T = float(mixed_delays(rng, 1)[0])
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        ewd = [(u, v, d[k]) for k, (u, v) in enumerate(edges)]
        at_b, _ = brute_forward(n, ewd, at_src)
        at = oracle.forward(n, m, in_ptr, in_src, d[perm], at_src)
        path = oracle.critical_path(n, m, in_ptr, in_src, d[perm], at, T).tolist()
        sinks = [v for v in range(n) if all(u != v for u, _ in edges)]
        exp_end = min(sinks, key=lambda v: (F32(F32(T) - at_b[v]), v))
        assert path[0] == exp_end, trial
        assert all(v != path[-1] for _, v in edges), trial          # ends at a source
        # some choice of parallel edges along the node path attains at_b[endpoint]
        hops = list(zip(path[1:], path[:-1]))                       # (u, v), source-ward
        choices = [[d[k] for k, (u, v) in enumerate(edges) if (u, v) == h] for h in hops]
        assert all(choices), trial
        best = None
        for combo in itertools.product(*choices[::-1]):             # source -> endpoint
            x = F32(at_src[path[-1]]) if at_src[path[-1]] != 0 else F32(0.0)
            for dk in combo:
                x = F32(x + F32(dk))
            best = x if best is None else max(best, x)
        assert best == at_b[path[0]], trial


def test_p11_critical_path_chain():
    g = hfgen.chain(3000, seed=5, relabel=True)
    src, dst = g.edges()
    nxt = np.full(g.n, -1, np.int64)
    nxt[src] = dst
    head = int(np.setdiff1d(np.arange(g.n), dst)[0])
    walk = [head]
    while nxt[walk[-1]] >= 0:
        walk.append(int(nxt[walk[-1]]))
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, np.ones(g.m, F32), None)
    path = oracle.critical_path(g.n, g.m, g.in_ptr, g.in_src, np.ones(g.m, F32), at, 1e6)
    assert path.tolist() == walk[::-1]     # the whole chain, endpoint first


def test_p11_critical_paths_top_k_integer():
    # top-K endpoints: the K sinks in (T - at, id) order computed in exact integers,
    # each traced with the integer greedy; -1 / empty past the number of sinks
    rng = np.random.default_rng(1103)
    for trial in range(300):
        n, edges = random_tiny_dag(rng, nmax=10, p=0.5)
        m = len(edges)
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        dst = np.repeat(np.arange(n), np.diff(in_ptr)).astype(np.int64)
        S = 3
        d_int = rng.integers(1, 5, size=(m, S))
        a_int = rng.integers(0, 3, size=n)
        T = rng.integers(20, 30, size=S)
        at = np.stack([oracle.forward(n, m, in_ptr, in_src, d_int[:, s].astype(F32),
                                      a_int.astype(F32)) for s in range(S)], axis=1)
        K = int(rng.integers(1, 6))
        ends, paths = oracle.critical_paths_k(n, m, in_ptr, in_src, d_int.astype(F32), at,
                                              T.astype(F32), K)
        src_l, dst_l = in_src.tolist(), dst.tolist()
        outdeg = np.bincount(in_src, minlength=n) if m else np.zeros(n, np.int64)
        for s in range(S):
            at_i = dfs_int_at(n, src_l, dst_l, d_int[:, s].tolist(), a_int.tolist())
            sinks = sorted((v for v in range(n) if outdeg[v] == 0),
                           key=lambda v: (int(T[s]) - at_i[v], v))
            for r in range(K):
                if r >= len(sinks):
                    assert ends[s, r] == -1 and len(paths[s][r]) == 0, (trial, s, r)
                    continue
                v = sinks[r]
                assert ends[s, r] == v, (trial, s, r)
                ins = [[] for _ in range(n)]
                for e in range(m):
                    ins[dst_l[e]].append(e)
                path = [v]
                while ins[v]:
                    e = min(e for e in ins[v] if at_i[src_l[e]] + d_int[e, s] == at_i[v])
                    v = src_l[e]
                    path.append(v)
                assert paths[s][r].tolist() == path, (trial, s, r)
        # K = 1 is the single worst path
        one = oracle.critical_paths(n, m, in_ptr, in_src, d_int.astype(F32), at, T.astype(F32))
        e1, p1 = oracle.critical_paths_k(n, m, in_ptr, in_src, d_int.astype(F32), at,
                                         T.astype(F32), 1)
        assert all(p1[s][0].tolist() == one[s].tolist() for s in range(S)), trial


# ---- P12: early (hold) mode -- min-plus forward, max-plus backward (NEXT-2, R18) ----
def test_p12_early_mode_bruteforce_tiny_dags():
    rng = np.random.default_rng(1203)
    for trial in range(800):
        n, edges = random_tiny_dag(rng)
        m = len(edges)
        d = mixed_delays(rng, m)
        at_src = mixed_delays(rng, n)
        T = float(mixed_delays(rng, 1)[0])
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        ewd = [(u, v, d[k]) for k, (u, v) in enumerate(edges)]
        at_b, _ = brute_forward(n, ewd, at_src, early=True)
        rat_b = brute_backward(n, ewd, T, early=True)
        at = oracle.forward(n, m, in_ptr, in_src, d[perm], at_src, early=True)
        assert np.array_equal(at.view(np.uint32), at_b.view(np.uint32)), trial
        rat, slack, wns = oracle.backward(n, m, in_ptr, in_src, d[perm], T, at, early=True)
        assert np.array_equal(rat.view(np.uint32), rat_b.view(np.uint32)), trial
        s_b = (at_b - rat_b).astype(F32)                       # hold slack = at - rat
        assert np.array_equal(slack.view(np.uint32), s_b.view(np.uint32)), trial
        assert wns == s_b.min()


def test_p12_early_late_duality():
    # min(x) = -max(-x) and round-to-nearest is sign-symmetric, so the early passes
    # on (d, at_src, T) are the negated late passes on (-d, -at_src, -T), exactly
    g = hfgen.config("C1")
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    a_e = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv, early=True)
    a_l = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, -g.delay, -g.at_src, lv)
    assert np.array_equal(a_e, -a_l)
    r_e, s_e, w_e = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, a_e, lv,
                                    early=True)
    r_l, s_l, w_l = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, -g.delay, -g.t_req, a_l, lv)
    assert np.array_equal(r_e, -r_l)
    assert np.array_equal(s_e, s_l)                            # fl(at - rat) = fl(rat_l - at_l)
    assert w_e == w_l
    # and the two modes differ on this graph (a dropped mode switch fails here)
    a_late = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
    assert (a_e < a_late).any() and (a_e <= a_late).all()


def test_p12_early_unit_delay_is_bfs_distance():
    g = hfgen.config("C3", 0.01)
    src, dst = g.edges()
    # shortest number of edges from any source: plain BFS fixpoint over the edge list
    indeg = np.bincount(dst, minlength=g.n)
    dist = np.where(indeg == 0, 0, np.iinfo(np.int64).max // 2)
    while True:
        cand = np.full(g.n, np.iinfo(np.int64).max // 2)
        np.minimum.at(cand, dst, dist[src] + 1)
        new = np.where(indeg == 0, 0, cand)
        if np.array_equal(new, dist):
            break
        dist = new
    at = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, np.ones(g.m, F32), None, early=True)
    assert np.array_equal(at, dist.astype(F32))


# ---- P13: greedy MIS (NEXT-4, reading R19) ----------------------------------------
def _lexfirst_mis_bruteforce(n, und_edges, key):
    """Enumerate all independent sets that are maximal; the lexicographically-first
    one visits vertices by increasing key and prefers membership."""
    order = sorted(range(n), key=lambda v: key[v])
    adj = [set() for _ in range(n)]
    for u, v in und_edges:
        adj[u].add(v)
        adj[v].add(u)
    best = None
    for mask in range(1 << n):
        S = [v for v in range(n) if mask >> v & 1]
        if any(u in adj[v] for v in S for u in S):
            continue
        if any(all(u not in adj[v] for u in S) for v in range(n) if not mask >> v & 1):
            continue                                          # not maximal
        vec = tuple(mask >> v & 1 for v in order)
        if best is None or vec > best[0]:
            best = (vec, mask)
    return np.array([best[1] >> v & 1 for v in range(n)], np.uint8)


def test_p13_mis_bruteforce_tiny():
    rng = np.random.default_rng(1313)
    for trial in range(300):
        n, edges = random_tiny_dag(rng, nmax=9, p=0.35)
        in_ptr, in_src, _ = csr_from_edges(n, edges)
        prio = rng.integers(0, 4, size=n).astype(np.int32)   # ties broken by id
        got = oracle.mis(n, len(edges), in_ptr, in_src, prio)
        exp = _lexfirst_mis_bruteforce(n, edges, [(int(prio[v]), v) for v in range(n)])
        assert np.array_equal(got, exp), trial


def test_p13_mis_characterisation_large():
    # independent, and every excluded vertex has an earlier (prio, id) neighbour in
    # the set: the two properties single out the lexicographically-first MIS
    g = hfgen.config("C3", 0.05)
    prio = np.random.default_rng(5).permutation(g.n).astype(np.int32)
    s = oracle.mis(g.n, g.m, g.in_ptr, g.in_src, prio)
    src, dst = g.edges()
    assert not (s[src] & s[dst]).any()                        # independent
    key = prio.astype(np.int64) * g.n + np.arange(g.n)
    earlier_in = np.zeros(g.n, bool)
    for a, b in ((src, dst), (dst, src)):                     # a's neighbour b
        hit = (key[b] < key[a]) & (s[b] == 1)
        earlier_in[a[hit]] = True
    assert np.array_equal(s == 0, earlier_in)


def test_p13_mis_closed_forms():
    k = 101
    in_ptr, in_src, _ = csr_from_edges(k, [(i, i + 1) for i in range(k - 1)])   # a path
    up = oracle.mis(k, k - 1, in_ptr, in_src, np.arange(k, dtype=np.int32))
    assert np.array_equal(np.nonzero(up)[0], np.arange(0, k, 2))
    down = oracle.mis(k, k - 1, in_ptr, in_src, np.arange(k, dtype=np.int32)[::-1].copy())
    assert np.array_equal(np.nonzero(down)[0], np.arange(k - 1, -1, -2)[::-1])
    star = [(0, i) for i in range(1, 20)]                      # centre 0
    in_ptr, in_src, _ = csr_from_edges(20, star)
    first = oracle.mis(20, 19, in_ptr, in_src, np.arange(20, dtype=np.int32))
    assert np.nonzero(first)[0].tolist() == [0]
    last = oracle.mis(20, 19, in_ptr, in_src, np.r_[99, np.arange(1, 20)].astype(np.int32))
    assert np.nonzero(last)[0].tolist() == list(range(1, 20))
