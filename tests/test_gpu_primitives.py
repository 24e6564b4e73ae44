"""GPU primitives used by ingest / levelize: the single-pass decoupled look-back scan
(through the hf_debug_scan test hook), checked against numpy on sizes that span one
tile, tile boundaries, ragged tails and repeated calls on one graph (epoch reuse)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2203_08395_b200 import build
    build.build()
    from paper_2203_08395_b200 import hf as _hf
    return _hf


def test_exclusive_scan_lookback(hf):
    import torch
    dev = torch.device("cuda:0")
    G = hf.hf_graph_create(2, 1, torch.tensor([0, 0, 1], dtype=torch.int32, device=dev),
                           torch.tensor([0], dtype=torch.int32, device=dev),
                           stream=torch.cuda.current_stream())
    lib = hf._lib
    lib.hf_debug_scan.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p]
    rng = np.random.default_rng(0)
    for n in [1, 5, 4095, 4096, 4097, 10001, 100000, 1500001, 3, 2500000, 8191, 123457]:
        a = rng.integers(0, 10, n).astype(np.int32)
        x = torch.from_numpy(a).to(dev)
        y = torch.empty_like(x)
        tot = torch.zeros(1, dtype=torch.int32, device=dev)
        assert lib.hf_debug_scan(G.handle, x.data_ptr(), y.data_ptr(), n, tot.data_ptr()) == 0
        ref = np.concatenate([[0], np.cumsum(a)[:-1]]).astype(np.int64)
        assert np.array_equal(y.cpu().numpy().astype(np.int64), ref), n
        assert int(tot.item()) == int(a.sum()), n
        # in place
        assert lib.hf_debug_scan(G.handle, x.data_ptr(), x.data_ptr(), n, None) == 0
        assert np.array_equal(x.cpu().numpy().astype(np.int64), ref), n
    G.close()
