"""GPU parity: libhf.so (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json:5): level / level_ptr / order exact; at, rat,
slack, wns 0 ULP (compared as uint32 bit patterns).  Sizes span several tiles and
ragged tails; full BASELINE sizes are covered with all outputs compared (the C
oracle finishes them in seconds).
"""
import os

import numpy as np
import pytest

import hfgen
import oracle
from helpers import csr_from_edges, load_golden, mixed_delays, random_tiny_dag, reach_from_cycles

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module")
def hf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2203_08395_b200 import build
    build.build()
    from paper_2203_08395_b200 import hf as _hf
    return _hf


def bits(x):
    return np.ascontiguousarray(x, dtype=F32).view(np.uint32)


def assert_bits_equal(a, b, what=""):
    a, b = np.asarray(a, F32), np.asarray(b, F32)
    assert a.shape == b.shape, what
    nan = np.isnan(a) & np.isnan(b)
    diff = (bits(a) != bits(b)) & ~nan
    if diff.any():
        i = np.argwhere(diff)[0]
        raise AssertionError(f"{what}: {diff.sum()} mismatches, first at {tuple(i)}: "
                             f"gpu={a[tuple(i)]!r} oracle={b[tuple(i)]!r}")


def gpu_single(hf, g_in_ptr, g_in_src, n, m, delay, at_src, T, fanout=None):
    kw = {}
    if fanout is not None:
        kw = dict(fanout_ptr=fanout[0], fanout_dst=fanout[1])
    G = hf.hf_graph_create(n, m, g_in_ptr, g_in_src, delay=delay, **kw)
    L, level, lptr, order = hf.levelize_np(G)
    at = np.zeros(max(n, 1), F32)
    hf.hf_propagate_forward(G, at_src, at)
    rat = np.zeros(max(n, 1), F32)
    slack = np.zeros(max(n, 1), F32)
    wns = np.zeros(1, F32)
    hf.hf_propagate_backward(G, T, at[:n], rat, slack, wns)
    G.close()
    return L, level, lptr, order, at[:n], rat[:n], slack[:n], wns[0]


def check_single(hf, n, m, in_ptr, in_src, delay, at_src, T, fanout=None):
    L, level, lptr, order, at, rat, slack, wns = gpu_single(hf, in_ptr, in_src, n, m, delay,
                                                            at_src, T, fanout)
    lv = oracle.levelize(n, m, in_ptr, in_src)
    assert L == lv.num_levels
    assert np.array_equal(level, lv.level)
    assert np.array_equal(lptr, lv.level_ptr)
    assert np.array_equal(order, lv.order)
    at_o = oracle.forward(n, m, in_ptr, in_src, delay, at_src, lv)
    assert_bits_equal(at, at_o, "at")
    rat_o, slack_o, wns_o = oracle.backward(n, m, in_ptr, in_src, delay, T, at_o, lv)
    assert_bits_equal(rat, rat_o, "rat")
    assert_bits_equal(slack, slack_o, "slack")
    assert_bits_equal(wns, wns_o, "wns")


# ---- the paper's worked graphs ------------------------------------------------
@pytest.mark.parametrize("fname", ["fig1_saxpy.txt", "fig5_dependency.txt"])
def test_golden_graphs(hf, fname):
    g = load_golden(fname)
    in_ptr, in_src, _ = csr_from_edges(g["n"], g["edge"])
    G = hf.hf_graph_create(g["n"], len(g["edge"]), in_ptr, in_src)
    L, level, lptr, order = hf.levelize_np(G)
    assert L == g["num_levels"]
    assert level.tolist() == g["level"]
    assert lptr.tolist() == g["level_ptr"]
    assert order.tolist() == g["order"]


# ---- configs at parity sizes and at full size ----------------------------------
@pytest.mark.parametrize("name,scale", [
    ("C1", 1.0), ("C3", 0.003), ("C3", 0.05), ("C2-random", 0.003), ("C5", 0.0005),
    ("C5", 0.01),
])
def test_config_single(hf, name, scale):
    g = hfgen.config(name, scale)
    check_single(hf, g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, g.t_req)


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_config_single_full(hf, name):
    g = hfgen.config(name)
    check_single(hf, g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, g.t_req)


@pytest.mark.parametrize("name", ["C2-chain", "C2-tree", "C2-random"])
def test_c2_levelize_full(hf, name):
    g = hfgen.config(name)
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=np.ones(g.m, F32))
    L, level, lptr, order = hf.levelize_np(G)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    assert L == lv.num_levels
    assert np.array_equal(level, lv.level)
    assert np.array_equal(lptr, lv.level_ptr)
    assert np.array_equal(order, lv.order)
    if g.level_label is not None:
        assert np.array_equal(level, g.level_label)
    # unit-delay forward: at == level exactly (P3)
    at = np.zeros(g.n, F32)
    hf.hf_propagate_forward(G, np.zeros(g.n, F32), at)
    assert np.array_equal(at, level.astype(F32))


# ---- tiny random DAGs, mixed-sign / mixed-magnitude delays, multi-edges --------
def test_tiny_random_dags(hf):
    rng = np.random.default_rng(100)
    for trial in range(150):
        n, edges = random_tiny_dag(rng, nmax=12)
        m = len(edges)
        d = mixed_delays(rng, m)
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        at_src = mixed_delays(rng, n)
        T = float(mixed_delays(rng, 1)[0])
        check_single(hf, n, m, in_ptr, in_src, d[perm], at_src, T)


def test_cycles_reported_with_unready_count(hf):
    rng = np.random.default_rng(5)
    seen = 0
    for trial in range(60):
        n, edges = random_tiny_dag(rng, nmax=10)
        if n < 2:
            continue
        edges.append((int(rng.integers(0, n)), int(rng.integers(0, n))))
        bad = reach_from_cycles(n, edges)
        in_ptr, in_src, _ = csr_from_edges(n, edges)
        G = hf.hf_graph_create(n, len(edges), in_ptr, in_src)
        if bad.any():
            seen += 1
            with pytest.raises(hf.HFError) as ei:
                hf.levelize_np(G)
            assert ei.value.status == hf.HF_ERR_CYCLE
            assert f"{int(bad.sum())} nodes never become ready" in str(ei.value)
            with pytest.raises(hf.HFError) as ei:
                hf.hf_propagate_forward(G, None, np.zeros(n, F32))
            assert ei.value.status == hf.HF_ERR_NOT_LEVELIZED
        else:
            hf.levelize_np(G)
    assert seen > 10


def test_cycle_in_large_graph(hf):
    g = hfgen.config("C3", 0.01)
    src, dst = g.edges()
    # back edge from a deep node to a shallow ancestor region + a long pure chain cycle
    deep = int(np.argmax(g.level_label))
    shallow = int(np.argmin(g.level_label))
    edges = list(zip(src.tolist(), dst.tolist())) + [(deep, shallow)]
    in_ptr, in_src, _ = csr_from_edges(g.n, edges)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.levelize(g.n, len(edges), in_ptr, in_src)
    G = hf.hf_graph_create(g.n, len(edges), in_ptr, in_src)
    with pytest.raises(hf.HFError) as ei:
        hf.levelize_np(G)
    assert f"{eo.value.unready} nodes never become ready" in str(ei.value)
    # pure in-degree-1 ring (pointer jumping must stop)
    ring = [(i, (i + 1) % 5000) for i in range(5000)] + [(5000, 5001)]
    ip, isrc, _ = csr_from_edges(5002, ring)
    G = hf.hf_graph_create(5002, len(ring), ip, isrc)
    with pytest.raises(hf.HFError) as ei:
        hf.levelize_np(G)
    assert "5000 nodes never become ready" in str(ei.value)


# ---- edge cases -------------------------------------------------------------------
def test_empty_graph(hf):
    G = hf.hf_graph_create(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32))
    L, level, lptr, order = hf.levelize_np(G)
    assert L == 0 and lptr.tolist() == [0]
    wns = np.zeros(1, F32)
    hf.hf_propagate_backward(G, 1.0, np.zeros(0, F32), np.zeros(1, F32), None, wns)
    assert np.isposinf(wns[0])


def test_isolated_nodes_and_negative_zero(hf):
    n = 1000
    in_ptr = np.zeros(n + 1, np.int32)
    at_src = np.where(np.arange(n) % 2 == 0, -0.0, np.arange(n)).astype(F32)
    check_single(hf, n, 0, in_ptr, np.zeros(0, np.int32), None, at_src, -0.0)


def test_multi_edges_hub_denormals(hf):
    rng = np.random.default_rng(3)
    n = 12_000
    edges = [(u, n - 1) for u in range(10_000)]                # 10k fan-in hub
    edges += [(0, 10_001)] * 5                                    # multi-edges
    edges += [(n - 1, 10_002 + k) for k in range(1000)]          # 1k fan-out
    m = len(edges)
    d = mixed_delays(rng, m)
    d[::7] = np.float32(1e-40)                                     # denormals
    d[1::11] = np.float32(-3e-39)
    d[2::13] = np.float32(-0.0)
    in_ptr, in_src, perm = csr_from_edges(n, edges)
    at_src = (mixed_delays(rng, n) * np.float32(1e-38)).astype(F32)   # denormal range
    check_single(hf, n, m, in_ptr, in_src, d[perm], at_src, 1e-38)


def test_invalid_inputs(hf):
    ip, isrc, _ = csr_from_edges(3, [(0, 1), (1, 2)])
    with pytest.raises(hf.HFError) as ei:
        hf.hf_graph_create(3, 2, ip, isrc, delay=np.array([1, np.nan], F32))
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    with pytest.raises(hf.HFError) as ei:
        hf.hf_graph_create(3, 2, ip, np.array([0, 3], np.int32))
    assert ei.value.status == hf.HF_ERR_BAD_CSR
    with pytest.raises(hf.HFError) as ei:
        hf.hf_graph_create(3, 2, np.array([0, 2, 1, 2], np.int32), isrc)
    assert ei.value.status == hf.HF_ERR_BAD_CSR
    G = hf.hf_graph_create(3, 2, ip, isrc)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_propagate_forward(G, None, np.zeros(3, F32))
    assert ei.value.status == hf.HF_ERR_NOT_LEVELIZED
    hf.levelize_np(G)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_run_batch(G, 2, np.array([[1, 2], [np.inf, 1]], F32), hf.HF_LAYOUT_MS,
                        np.ones(2, F32), None, np.zeros(2, F32))
    assert ei.value.status == hf.HF_ERR_INVALID_ARG


def test_caller_fanout_validated(hf):
    g = hfgen.config("C1", 0.2)
    op, od, oe = oracle.fanout(g.n, g.m, g.in_ptr, g.in_src)
    od2 = od.copy()
    rng = np.random.default_rng(1)
    for u in range(g.n):
        rng.shuffle(od2[op[u]:op[u + 1]])
    check_single(hf, g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, g.t_req, (op, od2))
    od3 = od2.copy()
    k = int(np.nonzero(np.diff(op))[0][3])
    od3[op[k]] = (od3[op[k]] + 1) % g.n
    with pytest.raises(hf.HFError) as ei:
        hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, op, od3, g.delay)
    assert ei.value.status == hf.HF_ERR_BAD_CSR


# ---- batched scenarios ---------------------------------------------------------------
def gpu_batch_device(hf, g, D_ms, T, s_local, want_at_rat=True):
    import torch
    dev = torch.device("cuda:0")
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    d = torch.from_numpy(np.ascontiguousarray(D_ms)).to(dev)
    t = torch.from_numpy(np.asarray(T, F32)).to(dev)
    a = torch.from_numpy(g.at_src).to(dev)
    w = torch.empty(s_local, dtype=torch.float32, device=dev)
    at = torch.empty(g.n * s_local, dtype=torch.float32, device=dev) if want_at_rat else None
    rat = torch.empty(g.n * s_local, dtype=torch.float32, device=dev) if want_at_rat else None
    hf.hf_run_batch(G, s_local, d, hf.HF_LAYOUT_MS, t, a, w, at=at, rat=rat)
    hf.hf_sync(G)
    out = (w.cpu().numpy(),
           at.cpu().numpy().reshape(g.n, s_local) if want_at_rat else None,
           rat.cpu().numpy().reshape(g.n, s_local) if want_at_rat else None)
    G.close()
    return out


@pytest.mark.parametrize("S", [1, 2, 3, 4, 8, 16, 24, 32, 48, 64, 96, 192])
def test_batch_small(hf, S):
    # every chunk shape: the single-chunk kernels (S = 1, 2, 4, 8, 16, 32, 64: one
    # lane-group width each), several chunks with a power-of-two count (S = 128 in the
    # schedule test below) and with three (S = 24, 48, 96, 192: the division locator)
    g = hfgen.config("C3", 0.004)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[::2] -= 3.5
    w, at, rat = gpu_batch_device(hf, g, D, T, S)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                                 want_at_rat=True)
    assert_bits_equal(at, ato, "at")
    assert_bits_equal(rat, rato, "rat")
    assert_bits_equal(w, wo, "wns")


@pytest.mark.parametrize("S", [64, 24])
def test_batch_long_rows(hf, S):
    # a graph with hubs (C3 at 5%: fan-out up to 91, 503 long backward rows cut into
    # parts): the partials of a long neighbour waited on as a group (single-chunk
    # kernel, S = 64) and one after the other (three chunks, S = 24)
    g = hfgen.config("C3", 0.05)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[1::3] += 1.25
    w, at, rat = gpu_batch_device(hf, g, D, T, S)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=8,
                                 want_at_rat=True)
    assert_bits_equal(at, ato, "at")
    assert_bits_equal(rat, rato, "rat")
    assert_bits_equal(w, wo, "wns")


@pytest.mark.parametrize("S", [3, 64])
def test_batch_concurrent_passes(hf, S, monkeypatch):
    # HF_CONCURRENT=1: forward and backward kernels resident side by side on two
    # streams, slack/WNS in a separate pass -- same bits as the oracle
    monkeypatch.setenv("HF_CONCURRENT", "1")
    g = hfgen.config("C3", 0.004)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[1::2] += 2.25
    w, at, rat = gpu_batch_device(hf, g, D, T, S)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                                 want_at_rat=True)
    assert_bits_equal(at, ato, "at")
    assert_bits_equal(rat, rato, "rat")
    assert_bits_equal(w, wo, "wns")


@pytest.mark.parametrize("knob,val", [("HF_GA", "1"), ("HF_POLL_ALL", "0"), ("HF_PREFILL", "1"),
                                      ("HF_BATCH_PLAIN", "1")])
@pytest.mark.parametrize("S", [64, 12])
def test_batch_kernel_variants(hf, knob, val, S, monkeypatch):
    # the measured-and-rejected variants kept as switches: cp.async
    # gathers into shared memory (HF_GA=1), one-lane polling (HF_POLL_ALL=0), the
    # forward kernel NaN-filling rat (HF_PREFILL=1), the batch as two plain passes
    # without the side stream (HF_BATCH_PLAIN=1)
    monkeypatch.setenv(knob, val)
    g = hfgen.config("C3", 0.004)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    w, at, rat = gpu_batch_device(hf, g, D, T, S)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                                 want_at_rat=True)
    assert_bits_equal(at, ato, "at")
    assert_bits_equal(rat, rato, "rat")
    assert_bits_equal(w, wo, "wns")


def test_batch_reuses_schedule_across_scenario_counts(hf):
    # one levelized graph, batches of S = 64, 128 (same task weight, new task bases),
    # 32 (new task weight: schedule rebuilt), 64 again, 1 (two index slots per lane):
    # every call bit-identical to the oracle
    import torch
    dev = torch.device("cuda:0")
    g = hfgen.config("C3", 0.004)
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    a = torch.from_numpy(g.at_src).to(dev)
    for S in (64, 128, 32, 64, 1):
        D = hfgen.scenario_delays(g, 0, S, "ms")
        T = np.full(S, g.t_req, F32)
        T[::5] -= 1.5
        d = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
        t = torch.from_numpy(T).to(dev)
        w = torch.empty(S, dtype=torch.float32, device=dev)
        at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
        rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
        hf.hf_run_batch(G, S, d, hf.HF_LAYOUT_MS, t, a, w, at=at, rat=rat)
        hf.hf_sync(G)
        wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms",
                                     threads=4, want_at_rat=True)
        assert_bits_equal(at.cpu().numpy().reshape(g.n, S), ato, f"at S={S}")
        assert_bits_equal(rat.cpu().numpy().reshape(g.n, S), rato, f"rat S={S}")
        assert_bits_equal(w.cpu().numpy(), wo, f"wns S={S}")
    G.close()


def test_analyze_one_call_host_api(hf):
    # hf_analyze = create + levelize + batch from host buffers (pinned and pageable),
    # same bits as the oracle; the kept graph is reusable; errors leave no graph
    import torch
    g = hfgen.config("C3", 0.004)
    S = 16
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[::3] += 0.75
    wo = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    for conv in (lambda a: a, pin):
        w = conv(np.zeros(S, F32))
        L, G = hf.hf_analyze(g.n, g.m, conv(g.in_ptr), conv(g.in_src), S, conv(D), conv(T),
                             conv(g.at_src), w, delay=conv(g.delay), keep_graph=True)
        assert_bits_equal(np.asarray(w), wo, "wns analyze")
        assert L == hf.hf_graph_info(G)[2]
        w2 = np.zeros(S, F32)
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, g.at_src, w2)
        assert_bits_equal(w2, wo, "wns reuse")
        G.close()
    # a 2-cycle: HF_ERR_CYCLE, nothing kept
    ptr = np.array([0, 1, 2], np.int32)
    src = np.array([1, 0], np.int32)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_analyze(2, 2, ptr, src, 1, np.zeros(2, F32), np.zeros(1, F32), None,
                      np.zeros(1, F32), keep_graph=True)
    assert ei.value.status == hf.HF_ERR_CYCLE


def test_batch_host_api_both_layouts(hf):
    g = hfgen.config("C1")
    S = 6
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    wo = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4)
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    hf.levelize_np(G)
    for layout, arr in ((hf.HF_LAYOUT_MS, D), (hf.HF_LAYOUT_SM, np.ascontiguousarray(D.T))):
        w = np.zeros(S, F32)
        hf.hf_run_batch(G, S, arr, layout, T, g.at_src, w)
        assert_bits_equal(w, wo, f"wns layout {layout}")


def test_batch_full_c4_and_shard_invariance(hf):
    """C4 at full size: all 64 worst slacks and the full at / rat matrices (every
    node, every scenario) exact; sharding into G = 2, 4, 8 blocks is bit-identical."""
    g = hfgen.config("C4")
    S = 64
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    w, at, rat = gpu_batch_device(hf, g, D, T, S)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms",
                                 threads=os.cpu_count() or 1, want_at_rat=True)
    assert_bits_equal(w, wo, "wns")
    assert_bits_equal(at, ato, "at (all 64 columns)")
    assert_bits_equal(rat, rato, "rat (all 64 columns)")
    del ato, rato
    for G_ in (2, 4, 8):
        parts = []
        for r in range(G_):
            lo, hi = r * S // G_, (r + 1) * S // G_
            parts.append(gpu_batch_device(hf, g, np.ascontiguousarray(D[:, lo:hi]), T[lo:hi],
                                          hi - lo, want_at_rat=False)[0])
        assert_bits_equal(np.concatenate(parts), w, f"shards G={G_}")


def test_batch_nccl_gather_single_rank(hf):
    """hf_run_batch with a 1-rank NCCL communicator: wns_all == wns_local."""
    import torch
    g = hfgen.config("C1")
    S = 8
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    uid = hf.hf_nccl_unique_id()
    comm = hf.hf_nccl_comm_init(uid, 0, 1, 0)
    try:
        dev = torch.device("cuda:0")
        G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay,
                               stream=torch.cuda.current_stream())
        hf.levelize_np(G)
        w = torch.empty(S, dtype=torch.float32, device=dev)
        wall = torch.empty(S, dtype=torch.float32, device=dev)
        hf.hf_run_batch(G, S, torch.from_numpy(D).to(dev), hf.HF_LAYOUT_MS,
                        torch.from_numpy(T).to(dev), torch.from_numpy(g.at_src).to(dev), w,
                        comm, wall)
        hf.hf_sync(G)
        wo = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4)
        assert_bits_equal(w.cpu().numpy(), wo, "wns_local")
        assert_bits_equal(wall.cpu().numpy(), wo, "wns_all")
        # host-pointer variant with the communicator
        wh = np.zeros(S, F32)
        wah = np.zeros(S, F32)
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, g.at_src, wh, comm, wah)
        assert_bits_equal(wah, wo, "wns_all host")
        G.close()
    finally:
        hf.hf_nccl_comm_destroy(comm)


# ---- NEXT-1: critical-path trace-back (reading R17) -----------------------------------
def test_critical_path_single_graph(hf):
    g = hfgen.config("C1")
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    L = hf.hf_levelize(G)
    at = np.zeros(g.n, F32)
    hf.hf_propagate_forward(G, g.at_src, at)
    path = hf.hf_critical_path(G, at, g.t_req, L)
    at_o = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src)
    assert_bits_equal(at, at_o, "at")
    exp = oracle.critical_path(g.n, g.m, g.in_ptr, g.in_src, g.delay, at_o, g.t_req)
    assert path.tolist() == exp.tolist()
    # an `at` that is not a forward result is rejected, not traced
    bad = at.copy()
    bad[exp[0]] += 1.0
    with pytest.raises(hf.HFError) as ei:
        hf.hf_critical_path(G, bad, g.t_req, L)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    G.close()


def test_critical_path_integer_ties_tiny(hf):
    rng = np.random.default_rng(311)
    for trial in range(60):
        n, edges = random_tiny_dag(rng, nmax=12, p=0.5)
        m = len(edges)
        in_ptr, in_src, _ = csr_from_edges(n, edges)
        d = rng.integers(1, 4, size=m).astype(F32)
        a_src = rng.integers(0, 3, size=n).astype(F32)
        G = hf.hf_graph_create(n, m, in_ptr, in_src, delay=d)
        L = hf.hf_levelize(G)
        at = np.zeros(max(n, 1), F32)
        hf.hf_propagate_forward(G, a_src, at)
        path = hf.hf_critical_path(G, at[:n], 30.0, max(L, 1))
        at_o = oracle.forward(n, m, in_ptr, in_src, d, a_src)
        exp = oracle.critical_path(n, m, in_ptr, in_src, d, at_o, 30.0)
        assert path.tolist() == exp.tolist(), trial
        G.close()


@pytest.mark.parametrize("name,scale,S", [("C3", 0.004, 8), ("C3", 0.004, 64), ("C3", 1.0, 4)])
def test_critical_path_batch_device(hf, name, scale, S):
    import torch
    dev = torch.device("cuda:0")
    g = hfgen.config(name, scale)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[1::3] -= 7.0
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    L = hf.hf_levelize(G)
    d = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
    t = torch.from_numpy(T).to(dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, d, hf.HF_LAYOUT_MS, t, torch.from_numpy(g.at_src).to(dev), w, at=at, rat=rat)
    path = torch.full((S, L), -7, dtype=torch.int32, device=dev)
    plen = torch.empty(S, dtype=torch.int32, device=dev)
    hf.hf_critical_path(G, at, t, L, path, plen, delays=d, s=S)
    hf.hf_sync(G)
    at_h = at.cpu().numpy().reshape(g.n, S)
    _, at_o, _ = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                              want_at_rat=True)
    assert_bits_equal(at_h, at_o, "at")
    exp = oracle.critical_paths(g.n, g.m, g.in_ptr, g.in_src, D, at_o, T, max_len=L)
    got_p, got_l = path.cpu().numpy(), plen.cpu().numpy()
    for s in range(S):
        assert got_l[s] == len(exp[s]), s
        assert got_p[s, :got_l[s]].tolist() == exp[s].tolist(), s
    G.close()


@pytest.mark.parametrize("name,scale,S,K", [("C3", 0.004, 8, 5), ("C3", 1.0, 4, 8),
                                           ("C3", 0.02, 2, 32), ("C1", 1.0, 130, 2),
                                           ("C1", 1.0, 3, 40), ("chain", 0, 2, 3)])
def test_critical_paths_top_k_device(hf, name, scale, S, K):
    # top-K endpoints per scenario (NEXT-1): endpoints, paths and lengths identical to
    # the oracle's; the chain has one sink (endpoint -1, length 0 past it).  K <= 32
    # takes the single selection (per-block lists + merge), K = 40 the per-rank passes
    import torch
    dev = torch.device("cuda:0")
    g = hfgen.chain(300, seed=3, relabel=True) if name == "chain" else hfgen.config(name, scale)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[1::2] -= 3.5
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    L = hf.hf_levelize(G)
    d = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
    t = torch.from_numpy(T).to(dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, d, hf.HF_LAYOUT_MS, t, torch.from_numpy(g.at_src).to(dev), w, at=at, rat=rat)
    ends = torch.full((S, K), -7, dtype=torch.int32, device=dev)
    path = torch.full((S, K, L), -7, dtype=torch.int32, device=dev)
    plen = torch.full((S, K), -7, dtype=torch.int32, device=dev)
    hf.hf_critical_paths(G, S, d, at, t, K, L, ends, path, plen)
    hf.hf_sync(G)
    at_h = at.cpu().numpy().reshape(g.n, S)
    e_o, p_o = oracle.critical_paths_k(g.n, g.m, g.in_ptr, g.in_src, D, at_h, T, K, max_len=L)
    got_e, got_p, got_l = ends.cpu().numpy(), path.cpu().numpy(), plen.cpu().numpy()
    assert np.array_equal(got_e, e_o)
    for s in range(S):
        for r in range(K):
            assert got_l[s, r] == len(p_o[s][r]), (s, r)
            assert got_p[s, r, :got_l[s, r]].tolist() == p_o[s][r].tolist(), (s, r)
    G.close()


# ---- NEXT-2: early (hold) mode (reading R18) --------------------------------------------
def _single_mode(hf, g, early, T):
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    hf.hf_graph_set_mode(G, hf.HF_MODE_EARLY if early else hf.HF_MODE_LATE)
    hf.hf_levelize(G)
    at = np.zeros(g.n, F32)
    hf.hf_propagate_forward(G, g.at_src, at)
    rat, slack, wns = np.zeros(g.n, F32), np.zeros(g.n, F32), np.zeros(1, F32)
    hf.hf_propagate_backward(G, T, at, rat, slack, wns)
    G.close()
    return at, rat, slack, wns[0]


@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C3", 0.01), ("C5", 0.002)])
def test_early_mode_single(hf, name, scale):
    g = hfgen.config(name, scale)
    T = np.float32(-3.75)   # hold requirement
    at, rat, slack, wns = _single_mode(hf, g, True, T)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    at_o = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv, early=True)
    rat_o, slack_o, wns_o = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, T, at_o, lv,
                                            early=True)
    assert_bits_equal(at, at_o, "at_early")
    assert_bits_equal(rat, rat_o, "rat_early")
    assert_bits_equal(slack, slack_o, "hold slack")
    assert_bits_equal(wns, wns_o, "hold wns")


def test_early_mode_tiny_and_switching(hf):
    rng = np.random.default_rng(1812)
    for trial in range(60):
        n, edges = random_tiny_dag(rng, nmax=12)
        m = len(edges)
        in_ptr, in_src, _ = csr_from_edges(n, edges)
        d = mixed_delays(rng, m)
        a_src = mixed_delays(rng, n)
        T = float(mixed_delays(rng, 1)[0])
        G = hf.hf_graph_create(n, m, in_ptr, in_src, delay=d)
        hf.hf_levelize(G)
        for early in (True, False, True):          # the mode switch takes effect per call
            hf.hf_graph_set_mode(G, hf.HF_MODE_EARLY if early else hf.HF_MODE_LATE)
            at = np.zeros(max(n, 1), F32)
            hf.hf_propagate_forward(G, a_src, at)
            rat, slack, wns = np.zeros(max(n, 1), F32), np.zeros(max(n, 1), F32), np.zeros(1, F32)
            hf.hf_propagate_backward(G, T, at[:n], rat, slack, wns)
            at_o = oracle.forward(n, m, in_ptr, in_src, d, a_src, early=early)
            rat_o, slack_o, wns_o = oracle.backward(n, m, in_ptr, in_src, d, T, at_o, early=early)
            assert_bits_equal(at[:n], at_o, f"at {trial} {early}")
            assert_bits_equal(rat[:n], rat_o, f"rat {trial} {early}")
            assert_bits_equal(slack[:n], slack_o, f"slack {trial} {early}")
            assert_bits_equal(wns[0], wns_o, f"wns {trial} {early}")
        G.close()


@pytest.mark.parametrize("S,concurrent", [(8, "0"), (64, "0"), (64, "1"), (3, "0")])
def test_early_mode_batch(hf, S, concurrent, monkeypatch):
    import torch
    monkeypatch.setenv("HF_CONCURRENT", concurrent)
    dev = torch.device("cuda:0")
    g = hfgen.config("C3", 0.004)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, -2.5, F32)
    T[::3] = 1.0
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_graph_set_mode(G, hf.HF_MODE_EARLY)
    hf.hf_levelize(G)
    d = torch.from_numpy(np.ascontiguousarray(D)).to(dev)
    t = torch.from_numpy(T).to(dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, d, hf.HF_LAYOUT_MS, t, torch.from_numpy(g.at_src).to(dev), w, at=at, rat=rat)
    hf.hf_sync(G)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                                 want_at_rat=True, early=True)
    assert_bits_equal(at.cpu().numpy().reshape(g.n, S), ato, "at_early")
    assert_bits_equal(rat.cpu().numpy().reshape(g.n, S), rato, "rat_early")
    assert_bits_equal(w.cpu().numpy(), wo, "hold wns")
    # the critical path is a late-mode notion
    with pytest.raises(hf.HFError) as ei:
        hf.hf_critical_path(G, np.zeros(g.n, F32), 0.0, 4)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    with pytest.raises(hf.HFError):
        hf.hf_graph_set_mode(G, 7)
    G.close()


# ---- NEXT-4: greedy MIS (reading R19) ------------------------------------------------
@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C3", 0.02), ("C3", 1.0), ("C2-random", 0.1),
                                        ("C5", 0.01)])
def test_mis_matches_oracle(hf, name, scale):
    g = hfgen.config(name, scale)
    prio = np.random.default_rng(44).permutation(g.n).astype(np.int32)
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src)
    got = hf.hf_mis(G, prio)
    G.close()
    exp = oracle.mis(g.n, g.m, g.in_ptr, g.in_src, prio)
    assert np.array_equal(got, exp), (name, int((got != exp).sum()))


def test_mis_ties_tiny_and_device_api(hf):
    import torch
    rng = np.random.default_rng(4404)
    for trial in range(80):
        n, edges = random_tiny_dag(rng, nmax=14, p=0.4)
        m = len(edges)
        in_ptr, in_src, _ = csr_from_edges(n, edges)
        prio = rng.integers(0, 3, size=n).astype(np.int32)      # many ties: broken by id
        G = hf.hf_graph_create(n, m, in_ptr, in_src)
        got = hf.hf_mis(G, prio)
        exp = oracle.mis(n, m, in_ptr, in_src, prio)
        assert np.array_equal(got, exp), trial
        G.close()
    g = hfgen.config("C1")
    dev = torch.device("cuda:0")
    prio = np.random.default_rng(7).permutation(g.n).astype(np.int32)
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), stream=torch.cuda.current_stream())
    out = torch.empty(g.n, dtype=torch.uint8, device=dev)
    hf.hf_mis(G, torch.from_numpy(prio).to(dev), out)
    hf.hf_sync(G)
    assert np.array_equal(out.cpu().numpy(), oracle.mis(g.n, g.m, g.in_ptr, g.in_src, prio))
    G.close()


@pytest.mark.parametrize("S", [256, 1024])
def test_view_sweep_full_c3(hf, S):
    """NEXT-3, the paper's view axis ("1024 timing reports",
    1113-1115): S DISTINCT delay sets (hfgen keys every scenario by its global id) on
    the full C3 graph in one batch.  Every scenario's worst slack is exact; at / rat
    are exact for every node of the last 64-column chunk (the chunk the kernels
    process last at the highest column offset)."""
    import torch
    dev = torch.device("cuda:0")
    g = hfgen.config("C3")
    B = 64
    T = np.full(S, g.t_req, F32)
    T[1::3] -= 2.5
    T[2::7] += 11.0
    d = torch.empty((g.m, S), dtype=torch.float32, device=dev)
    wo = np.empty(S, F32)
    chunk = S // B - 1
    for b in range(S // B):
        Db = hfgen.scenario_delays(g, b * B, (b + 1) * B, "ms")
        d[:, b * B:(b + 1) * B].copy_(torch.from_numpy(Db))
        res = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, Db, T[b * B:(b + 1) * B], g.at_src, "ms",
                           threads=os.cpu_count() or 1, want_at_rat=(b == chunk))
        if b == chunk:
            wo[b * B:(b + 1) * B], ato, rato = res
        else:
            wo[b * B:(b + 1) * B] = res
        del Db
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    at = torch.empty((g.n, S), dtype=torch.float32, device=dev)
    rat = torch.empty((g.n, S), dtype=torch.float32, device=dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, d, hf.HF_LAYOUT_MS, torch.from_numpy(T).to(dev),
                    torch.from_numpy(g.at_src).to(dev), w, at=at, rat=rat)
    hf.hf_sync(G)
    G.close()
    assert_bits_equal(w.cpu().numpy(), wo, f"wns S={S}")
    c0 = chunk * B
    assert_bits_equal(at[:, c0:c0 + B].cpu().numpy(), ato, f"at[:, {c0}:{c0 + B}]")
    assert_bits_equal(rat[:, c0:c0 + B].cpu().numpy(), rato, f"rat[:, {c0}:{c0 + B}]")


def test_batch_scratch_size_changes_keep_the_kernel_launchable(hf):
    """One kernel, two shared-memory sizes, in the order that used to fail: S = 128
    (larger scratch), then S = 64 for the first time (smaller), then S = 128 again --
    the dynamic shared-memory limit is only ever raised (common.cuh ensure_dyn_smem),
    so every call launches and stays bit-exact."""
    import torch
    dev = torch.device("cuda:0")
    g = hfgen.config("C3", 0.004)
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    a = torch.from_numpy(g.at_src).to(dev)
    for S in (128, 64, 128, 64):
        D = hfgen.scenario_delays(g, 0, S, "ms")
        T = np.full(S, g.t_req, F32)
        w = torch.empty(S, dtype=torch.float32, device=dev)
        hf.hf_run_batch(G, S, torch.from_numpy(D).to(dev), hf.HF_LAYOUT_MS, torch.from_numpy(T).to(dev),
                        a, w)
        hf.hf_sync(G)
        wo = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4)
        assert_bits_equal(w.cpu().numpy(), wo, f"wns S={S}")
    G.close()
