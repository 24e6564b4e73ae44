"""GPU parity of the level-synchronous ("wide") passes (wide.cu), forced on with
HF_WIDE=1 for graphs of every shape (by default they run only when a level holds
>= 32768 nodes on average, e.g. full C5).  Same bar as every propagation path:
at, rat, slack, wns 0 ULP against the oracle (BASELINE.json:5).
"""
import numpy as np
import pytest

import hfgen
import oracle
from helpers import csr_from_edges, mixed_delays, random_tiny_dag
from test_gpu_parity import assert_bits_equal, check_single, gpu_batch_device

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600, method="thread")]
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


# S = 1 runs k_wide3 (edge units, ordered-int accumulation in place) by default; the
# staged-tile k_wide4 (HF_WIDE4=1), the warp-unit kernel k_wide1 (HF_WIDE3=0) and the
# row-range kernel k_wide2 (HF_WIDE2=1) stay under test
KERNELS = {"w4": {"HF_WIDE3": "1", "HF_WIDE4": "1"}, "w3": {"HF_WIDE3": "1", "HF_WIDE4": "0"},
           "w1": {"HF_WIDE3": "0", "HF_WIDE2": "0"}, "w2": {"HF_WIDE3": "0", "HF_WIDE2": "1"}}


def use_kernel(monkeypatch, name):
    for k, v in KERNELS[name].items():
        monkeypatch.setenv(k, v)


@pytest.mark.parametrize("w2", ["w4", "w3", "w1", "w2"])
@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C3", 0.05), ("C2-random", 0.01),
                                        ("C5", 0.01), ("C5", 0.1)])
def test_wide_single(hf, name, scale, w2, monkeypatch):
    monkeypatch.setenv("HF_WIDE", "1")
    use_kernel(monkeypatch, w2)
    g = hfgen.config(name, scale)
    check_single(hf, g.n, g.m, g.in_ptr, g.in_src, g.delay, g.at_src, g.t_req)


@pytest.mark.parametrize("w2", ["w4", "w3", "w1", "w2"])
def test_wide_tiny_random_dags(hf, w2, monkeypatch):
    monkeypatch.setenv("HF_WIDE", "1")
    use_kernel(monkeypatch, w2)
    rng = np.random.default_rng(2203)
    for trial in range(80):
        n, edges = random_tiny_dag(rng, nmax=12)
        m = len(edges)
        in_ptr, in_src, perm = csr_from_edges(n, edges)
        d = mixed_delays(rng, m)
        check_single(hf, n, m, in_ptr, in_src, d[perm], mixed_delays(rng, n),
                     float(mixed_delays(rng, 1)[0]))


@pytest.mark.parametrize("w2", ["w4", "w3", "w1", "w2"])
def test_wide_hub_fan_in(hf, w2, monkeypatch):
    """One node with 10^4 predecessors (C5's planted hub): k_wide1 folds its slices by
    atomics into one slot and its consumers read the slot; k_wide2 keeps the row in
    one range (its 10^4 edges streamed through the shared accumulator); k_wide3 spans
    313 edge units whose pieces meet in ordered-int atomics."""
    monkeypatch.setenv("HF_WIDE", "1")
    use_kernel(monkeypatch, w2)
    rng = np.random.default_rng(7)
    k = 10000
    edges = [(i, k) for i in range(k)] + [(k, k + 1), (k, k + 2), (3, k + 2)]
    n = k + 3
    in_ptr, in_src, perm = csr_from_edges(n, edges)
    d = mixed_delays(rng, len(edges))
    check_single(hf, n, len(edges), in_ptr, in_src, d[perm], mixed_delays(rng, n), 1e3)


@pytest.mark.parametrize("S", [1, 3, 8, 64])
def test_wide_batch(hf, S, monkeypatch):
    monkeypatch.setenv("HF_WIDE", "1")
    g = hfgen.config("C5", 0.005)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, g.t_req, F32)
    T[::2] -= 1.5
    w, at, rat = gpu_batch_device(hf, g, D, T, S)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=8,
                                 want_at_rat=True)
    assert_bits_equal(at, ato, "at")
    assert_bits_equal(rat, rato, "rat")
    assert_bits_equal(w, wo, "wns")


@pytest.mark.parametrize("S", [1, 8])
def test_wide_early_mode(hf, S, monkeypatch):
    import torch
    monkeypatch.setenv("HF_WIDE", "1")
    dev = torch.device("cuda:0")
    g = hfgen.config("C5", 0.002)
    D = hfgen.scenario_delays(g, 0, S, "ms")
    T = np.full(S, -2.5, F32)
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_graph_set_mode(G, hf.HF_MODE_EARLY)
    hf.hf_levelize(G)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, torch.from_numpy(D).to(dev), hf.HF_LAYOUT_MS, torch.from_numpy(T).to(dev),
                    torch.from_numpy(g.at_src).to(dev), w, at=at, rat=rat)
    hf.hf_sync(G)
    wo, ato, rato = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=4,
                                 want_at_rat=True, early=True)
    assert_bits_equal(at.cpu().numpy().reshape(g.n, S), ato, "at_early")
    assert_bits_equal(rat.cpu().numpy().reshape(g.n, S), rato, "rat_early")
    assert_bits_equal(w.cpu().numpy(), wo, "hold wns")
    G.close()


def test_wide_nonfinite_terminates(hf, monkeypatch):
    monkeypatch.setenv("HF_WIDE", "1")
    g = hfgen.config("C5", 0.002)
    S = 4
    D = hfgen.scenario_delays(g, 0, S, "ms").copy()
    D[g.m // 2, 1] = np.nan
    G = hf.hf_graph_create(g.n, g.m, g.in_ptr, g.in_src, delay=g.delay)
    hf.hf_levelize(G)
    with pytest.raises(hf.HFError) as ei:
        hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, np.full(S, g.t_req, F32), g.at_src,
                        np.zeros(S, F32))
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    G.close()
