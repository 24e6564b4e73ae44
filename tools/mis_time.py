"""NEXT-4 timing: greedy MIS (hf_mis_d) on C3 / C5 / C2-random with random priorities;
CUDA events around the call (median of 5 after a warm-up), oracle time beside it."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hfgen  # noqa: E402
import oracle  # noqa: E402
from paper_2203_08395_b200 import hf  # noqa: E402

dev = torch.device("cuda:0")
for name in sys.argv[1:] or ["C3", "C2-random", "C5"]:
    g = hfgen.config(name)
    prio = np.random.default_rng(1).permutation(g.n).astype(np.int32)
    st = torch.cuda.current_stream()
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev), stream=st)
    p = torch.from_numpy(prio).to(dev)
    out = torch.empty(g.n, dtype=torch.uint8, device=dev)
    ts = []
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        hf.hf_mis(G, p, out)
        e1.record(st)
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    t0 = time.perf_counter()
    exp = oracle.mis(g.n, g.m, g.in_ptr, g.in_src, prio)
    t_cpu = time.perf_counter() - t0
    ok = np.array_equal(out.cpu().numpy(), exp)
    ms = float(np.median(ts))
    print(f"{name}: n={g.n} m={g.m} |MIS|={int(exp.sum())} gpu {ms:.3f} ms "
          f"({2 * g.m / ms / 1e6:.2f} G edge-visits/s); oracle 1 core {t_cpu * 1e3:.0f} ms; "
          f"identical={ok}", flush=True)
    G.close()
