"""GPU: rejected inputs terminate and report, scenario counts beyond one block.

* Non-finite inputs (reading R9, hf.h conventions; "never aborts"):
  a NaN scenario delay on the only fan-in edge of a node, a NaN required time
  and a NaN source arrival time each return HF_ERR_INVALID_ARG through every
  entry point that can receive them -- and the call returns at all: the
  propagation kernels treat NaN as "not yet computed", so an unguarded NaN row
  would be polled forever.  Each test carries a timeout so a regression fails
  instead of hanging the suite.  After the error the graph is still usable and
  bit-identical to the oracle.
* Scenario counts whose rows are wider than one thread block (S/V > 256 in the
  long-row finalisation and the slack epilogue): S = 257 (V = 1), 514 (V = 2),
  2048 (V = 4) on a graph with long rows, all at/rat/wns 0 ULP against the oracle.
"""
import os

import numpy as np
import pytest

import hfgen
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300, method="thread")]
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


@pytest.fixture(scope="module")
def g():
    return hfgen.config("C3", 0.004)


def bits(x):
    return np.ascontiguousarray(x, dtype=F32).view(np.uint32)


def indeg1_edge(g):
    """(node, edge id) of a node whose only fan-in edge is that edge."""
    deg = np.diff(g.in_ptr)
    v = int(np.nonzero(deg == 1)[0][len(np.nonzero(deg == 1)[0]) // 2])
    return v, int(g.in_ptr[v])


def a_source(g):
    return int(np.nonzero(np.diff(g.in_ptr) == 0)[0][0])


def bad_inputs(g, S, kind):
    D = hfgen.scenario_delays(g, 0, S, "ms").copy()
    T = np.full(S, g.t_req, F32)
    at_src = g.at_src.copy()
    if kind == "delay":
        _, e = indeg1_edge(g)
        D[e, S // 2] = np.nan
    elif kind == "t_req":
        T[S - 1] = np.nan
    elif kind == "at_src":
        at_src[a_source(g)] = np.nan
    elif kind == "inf_pair":   # opposite-sign infinities on one path
        _, e = indeg1_edge(g)
        D[e, 0] = np.inf
        D[(e + 1) % g.m, 0] = -np.inf
    return D, T, at_src


def check_valid_after(hf, G, g, S, run):
    """The same graph, valid inputs: bit-identical to the oracle."""
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    w = run(G, D, T, g.at_src)
    wo, _, _ = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                            want_at_rat=True)
    assert np.array_equal(bits(w), bits(wo))


KINDS = ["delay", "t_req", "at_src", "inf_pair"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("S", [1, 8, 64])
def test_nonfinite_run_batch_host(hf, g, kind, S):
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    hf.hf_levelize(G)
    D, T, a = bad_inputs(g, S, kind)
    w = np.zeros(S, F32)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, a, w)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG

    def run(G, D, T, a):
        w = np.zeros(S, F32)
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, a, w)
        return w
    check_valid_after(hf, G, g, S, run)
    G.close()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("S", [1, 64])
def test_nonfinite_run_batch_device(hf, g, kind, S):
    import torch
    dev = torch.device("cuda:0")
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev),
                           delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    D, T, a = bad_inputs(g, S, kind)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, torch.from_numpy(D).to(dev), hf.HF_LAYOUT_MS,
                    torch.from_numpy(T).to(dev), torch.from_numpy(a).to(dev), w)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_sync(G)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    hf.hf_sync(G)   # the error was cleared by the report

    def run(G, D, T, a):
        w = torch.empty(S, dtype=torch.float32, device=dev)
        hf.hf_run_batch(G, S, torch.from_numpy(np.ascontiguousarray(D)).to(dev),
                        hf.HF_LAYOUT_MS, torch.from_numpy(T).to(dev), torch.from_numpy(a).to(dev),
                        w)
        hf.hf_sync(G)
        return w.cpu().numpy()
    check_valid_after(hf, G, g, S, run)
    G.close()


@pytest.mark.parametrize("kind", KINDS)
def test_nonfinite_analyze(hf, g, kind):
    S = 16
    D, T, a = bad_inputs(g, S, kind)
    w = np.zeros(S, F32)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_analyze(g.n, g.m, g.in_ptr, g.in_src, S, D, T, a, w, delay=g.delay)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    # a following valid call on the same device is unaffected
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    hf.hf_analyze(g.n, g.m, g.in_ptr, g.in_src, S, D, T, g.at_src, w, delay=g.delay)
    wo, _, _ = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                            want_at_rat=True)
    assert np.array_equal(bits(w), bits(wo))


def test_nonfinite_single_graph_at_src(hf, g):
    import torch
    dev = torch.device("cuda:0")
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay,
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    a = g.at_src.copy()
    a[a_source(g)] = np.nan
    at = torch.empty(g.n, dtype=torch.float32, device=dev)
    hf.hf_propagate_forward(G, torch.from_numpy(a).to(dev), at)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_sync(G)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    with pytest.raises(hf.HFError) as ei:   # host variant: checked on the host
        hf.hf_propagate_forward(G, a, np.zeros(g.n, F32))
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    # a NaN `at` given to the backward pass only poisons the slack, never a polled row
    rat = torch.empty(g.n, dtype=torch.float32, device=dev)
    at_bad = torch.full((g.n,), float("nan"), device=dev)
    hf.hf_propagate_backward(G, float(g.t_req), at_bad, rat)
    hf.hf_sync(G)
    lv = oracle.levelize(g.n, g.m, g.in_ptr, g.in_src)
    at_o = oracle.forward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, lv)
    rat_o, _, _ = oracle.backward(g.n, g.m, g.in_ptr, g.in_src, g.delay, g.t_req, at_o, lv)
    assert np.array_equal(bits(rat.cpu().numpy()), bits(rat_o))
    G.close()


def test_output_arrays_checked(hf, g):
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    hf.hf_levelize(G)
    with pytest.raises(TypeError):
        hf.hf_propagate_forward(G, None, np.zeros(g.n))            # float64
    with pytest.raises(ValueError):
        hf.hf_propagate_forward(G, None, np.zeros(g.n - 1, F32))   # short
    with pytest.raises(ValueError):
        hf.hf_run_batch(G, 4, hfgen.scenario_delays(g, 0, 4, "ms"), hf.HF_LAYOUT_MS,
                        np.ones(4, F32), None, np.zeros(3, F32))
    G.close()


def test_scenario_count_limits(hf, g):
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    hf.hf_levelize(G)
    for S in (0, 8193):
        with pytest.raises(hf.HFError) as ei:
            hf.hf_run_batch(G, S, np.zeros(max(S, 1) * g.m, F32), hf.HF_LAYOUT_MS,
                            np.ones(max(S, 1), F32), None, np.zeros(max(S, 1), F32))
        assert ei.value.status == hf.HF_ERR_INVALID_ARG
    G.close()


@pytest.mark.parametrize("S", [257, 514, 2048])
@pytest.mark.parametrize("concurrent", ["0", "1"])
def test_wide_rows_finalisation(hf, g, S, concurrent, monkeypatch):
    """Long rows (degree > 8) finalised with S/V > 256 column vectors per row."""
    import torch
    monkeypatch.setenv("HF_CONCURRENT", concurrent)
    assert np.diff(oracle.fanout(g.n, g.m, g.in_ptr, g.in_src)[0]).max() > 8
    dev = torch.device("cuda:0")
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay,
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[::3] -= 7.25
    w = torch.empty(S, dtype=torch.float32, device=dev)
    at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, torch.from_numpy(D).to(dev), hf.HF_LAYOUT_MS, torch.from_numpy(T).to(dev),
                    torch.from_numpy(g.at_src).to(dev), w, at=at, rat=rat)
    hf.hf_sync(G)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=8,
                                 want_at_rat=True)
    assert np.array_equal(bits(at.cpu().numpy().reshape(g.n, S)), bits(ato))
    assert np.array_equal(bits(rat.cpu().numpy().reshape(g.n, S)), bits(rato))
    assert np.array_equal(bits(w.cpu().numpy()), bits(wo))
    G.close()


def test_watchdog_turns_a_stuck_wait_into_an_error(hf, monkeypatch):
    """HF_WATCHDOG_SPINS=1: every dataflow wait gives up after one poll round, as a
    schedule bug would after seconds -- the call must return HF_ERR_CUDA ('watchdog')
    instead of hanging, and the next call on the same graph must be clean."""
    import torch
    dev = torch.device("cuda:0")
    g = hfgen.config("C3")
    S = 64
    D = torch.from_numpy(hfgen.scenario_delays(g, 0, S, "ms")).to(dev)
    T = torch.full((S,), float(g.t_req), dtype=torch.float32, device=dev)
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    at_src = torch.from_numpy(g.at_src).to(dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    monkeypatch.setenv("HF_WATCHDOG_SPINS", "1")
    with pytest.raises(hf.HFError) as ei:
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
        hf.hf_sync(G)
    assert ei.value.status == hf.HF_ERR_CUDA and "watchdog" in str(ei.value)
    monkeypatch.delenv("HF_WATCHDOG_SPINS")
    hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
    hf.hf_sync(G)
    wo = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D.cpu().numpy(), T.cpu().numpy(), g.at_src,
                      "ms", threads=os.cpu_count() or 1)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), wo.view(np.uint32))
    G.close()
