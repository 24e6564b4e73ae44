"""Strong-scaling table on ONE B200 (BASELINE.json:10): C4's 64
scenarios split over G GPUs leave S_local = 64 / G scenarios per GPU; the per-GPU
propagation phase at S_local bounds the G-GPU step (the graph is replicated, the
only exchange is the 4-byte-per-scenario worst-slack all-gather).  For S_local = 64,
32, 16, 8 this times the batch phase (CUDA events inside the library, L2 flushed,
median of --reps) back to back and with HF_CONCURRENT=1 (forward and backward
kernels resident side by side), and prints the projected speed-up T(64) / T(S_local)
at G = 64 / S_local (gather not included: a few us).

    python tools/strong_table.py [--reps 7]
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
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = hfgen.config("C4")
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev),
                           delay=torch.from_numpy(g.delay).to(dev), stream=torch.cuda.current_stream())
    hf.hf_profile_enable(G, True)
    hf.hf_levelize(G)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    at_src = torch.from_numpy(g.at_src).to(dev)
    D64 = torch.from_numpy(hfgen.scenario_delays(g, 0, 64, "ms")).to(dev)
    rows = []
    base = os.environ.copy()
    for S in (64, 32, 16, 8):
        D = D64[:, :S].contiguous()   # rank 0's block: global scenarios 0 .. S-1
        T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
        w = torch.empty(S, dtype=torch.float32, device=dev)
        res = {}
        for conc in ("0", "1"):
            os.environ["HF_CONCURRENT"] = conc
            ph = []
            for r in range(a.reps + 1):
                flush.fill_(1.0)
                hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
                p = hf.hf_profile_read_batch(G)
                if r:
                    ph.append(p)
            res[conc] = float(np.median(ph))
        os.environ.clear()
        os.environ.update(base)
        rows.append((S, res["0"], res["1"]))
    t1 = min(rows[0][1], rows[0][2])
    print(f"C4 graph n={g.n} m={g.m}; batch phase (fills + task bases + forward + backward + WNS) "
          f"per GPU, median of {a.reps}")
    print(f"{'S_local':>7} {'G':>3} {'phase ms':>9} {'concurrent ms':>14} {'best ms':>8} "
          f"{'T1/T(S_local)':>14}")
    for S, p0, p1 in rows:
        b = min(p0, p1)
        print(f"{S:7d} {64 // S:3d} {p0:9.3f} {p1:14.3f} {b:8.3f} {t1 / b:14.2f}")
    G.close()


if __name__ == "__main__":
    main()
