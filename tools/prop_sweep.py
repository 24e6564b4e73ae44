"""Propagation-only timing sweep: fwd/bwd device ms per pass for several S.

    python tools/prop_sweep.py [--config C3] [--S 1,8,64,256] [--reps 5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hfgen  # noqa: E402
from paper_2203_08395_b200 import hf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--S", default="1,8,64,256")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--once", action="store_true", help="one batch per S (for ncu)")
    ap.add_argument("--single", action="store_true",
                    help="also time the single-graph calls (graph delays, S = 1)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = hfgen.config(a.config)
    st = torch.cuda.current_stream()
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev),
                           delay=torch.from_numpy(g.delay).to(dev), stream=st)
    hf.hf_profile_enable(G, True)
    L = hf.hf_levelize(G)
    lev_ms = hf.hf_profile_read(G)[0]
    print(f"{a.config}: n={g.n} m={g.m} L={L} levelize {lev_ms:.3f} ms")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    at_src = torch.from_numpy(g.at_src).to(dev)
    if a.single:
        at = torch.empty(g.n, dtype=torch.float32, device=dev)
        rat = torch.empty(g.n, dtype=torch.float32, device=dev)
        w1 = torch.empty(1, dtype=torch.float32, device=dev)
        f, b = [], []
        for r in range(1 if a.once else a.reps + 1):
            flush.fill_(1.0)
            hf.hf_propagate_forward(G, at_src, at)
            hf.hf_propagate_backward(G, float(g.t_req), at, rat, None, w1)
            _, fm, bm, _ = hf.hf_profile_read(G)
            if r > 0 or a.once:
                f.append(fm)
                b.append(bm)
        fm, bm = float(np.median(f)), float(np.median(b))
        nb_f = 4 * (g.n + 1) + 8 * g.m + (4 * g.m + 8 * g.n)
        nb_b = 4 * (g.n + 1) + 12 * g.m + (4 * g.m + 12 * g.n) + 4
        print(f"single fwd {fm:8.3f} ms ({nb_f / fm / 1e6:7.1f} GB/s)  bwd {bm:8.3f} ms "
              f"({nb_b / bm / 1e6:7.1f} GB/s)  f+b {(nb_f + nb_b) / (fm + bm) / 1e6:7.1f} GB/s  "
              f"edges/s {2 * g.m / ((fm + bm) * 1e-3):.3e}")
    for S in [int(x) for x in a.S.split(",") if x]:
        D = torch.from_numpy(hfgen.scenario_delays(g, 0, S, "ms")).to(dev)
        T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
        w = torch.empty(S, dtype=torch.float32, device=dev)
        f, b = [], []
        for r in range(1 if a.once else a.reps + 1):
            flush.fill_(1.0)
            hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
            _, fm, bm, _ = hf.hf_profile_read(G)
            if r > 0 or a.once:
                f.append(fm)
                b.append(bm)
        fm, bm = float(np.median(f)), float(np.median(b))
        nb_f = 4 * (g.n + 1) + 8 * g.m + S * (4 * g.m + 8 * g.n)
        nb_b = 4 * (g.n + 1) + 12 * g.m + S * (4 * g.m + 12 * g.n) + 4 * S
        print(f"S={S:5d} fwd {fm:8.3f} ms ({nb_f / fm / 1e6:7.1f} GB/s, {fm * 1e3 / L:6.2f} us/level)"
              f"  bwd {bm:8.3f} ms ({nb_b / bm / 1e6:7.1f} GB/s)  "
              f"edges/s {2 * g.m * S / ((fm + bm) * 1e-3):.3e}")


if __name__ == "__main__":
    main()
