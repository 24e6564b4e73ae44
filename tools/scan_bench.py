"""Time the library's exclusive scan (hf_debug_scan hook) on n = 1.5M int32."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_08395_b200 import hf  # noqa: E402

dev = torch.device("cuda:0")
G = hf.hf_graph_create(2, 1, torch.tensor([0, 0, 1], dtype=torch.int32, device=dev),
                       torch.tensor([0], dtype=torch.int32, device=dev),
                       stream=torch.cuda.current_stream())
lib = hf._lib
lib.hf_debug_scan.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p]
for n in (201, 1_500_001, 10_000_001):
    x = torch.randint(0, 9, (n,), dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    ts = []
    for r in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.hf_debug_scan(G.handle, x.data_ptr(), y.data_ptr(), n, None)
        e1.record()
        e1.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ok = torch.equal(y[1:].long(), torch.cumsum(x.long(), 0)[:-1]) and int(y[0]) == 0
    print(f"n={n}: {np.median(ts):.1f} us (incl. the hook's stream sync) ok={ok}")
G.close()
