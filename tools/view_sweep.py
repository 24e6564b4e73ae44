"""NEXT-3: paper-scale view sweep (PAPER.md:999-1001,
1113-1115 -- the paper's problem-size axis is the number of timing views).

One C3 graph (1.5M pins / 2.5M arcs), levelized once; for every view count S the
batch (forward + backward + slack + worst slack over S delay sets) is timed with
CUDA events (median of --reps after one warm-up, L2 flushed before each rep).
Delay sets: S DISTINCT what-if sets (hfgen keys each scenario by its global id),
generated on the host in blocks of 64 and uploaded into the columns of one
[m][S] device array; the same S-view batches are parity-tested against the oracle
at S = 256 and 1024 (tests/test_gpu_parity.py::test_view_sweep_full_c3).

    python tools/view_sweep.py [--S 32,64,128,256,512,1024] [--reps 3]
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
    ap.add_argument("--S", default="32,64,128,256,512,1024")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = hfgen.config(a.config)
    st = torch.cuda.current_stream()
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev),
                           delay=torch.from_numpy(g.delay).to(dev), stream=st)
    hf.hf_profile_enable(G, True)
    L = hf.hf_levelize(G)
    at_src = torch.from_numpy(g.at_src).to(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    peak = 6550.4
    try:
        import json
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
            os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    print(f"{a.config}: n={g.n} m={g.m} L={L}; HBM peak {peak:.0f} GB/s")
    print(f"{'S':>5} {'fwd ms':>8} {'bwd ms':>8} {'phase ms':>9} {'GB/s (kern)':>12} {'frac':>6} "
          f"{'edges/s (kern)':>15} {'GB resident':>12}")
    for S in [int(x) for x in a.S.split(",")]:
        D = torch.empty((g.m, S), dtype=torch.float32, device=dev)
        for b0 in range(0, S, 64):
            b1 = min(S, b0 + 64)
            D[:, b0:b1].copy_(torch.from_numpy(hfgen.scenario_delays(g, b0, b1, "ms")))
        T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
        w = torch.empty(S, dtype=torch.float32, device=dev)
        f, b, ph = [], [], []
        for r in range(a.reps + 1):
            flush.fill_(1.0)
            hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
            _, fm, bm, _ = hf.hf_profile_read(G)
            pm = hf.hf_profile_read_batch(G)
            if r:
                f.append(fm)
                b.append(bm)
                ph.append(pm)
        fm, bm, pm = (float(np.median(x)) for x in (f, b, ph))
        nb_f = 4 * (g.n + 1) + 8 * g.m + S * (4 * g.m + 8 * g.n)
        nb_b = 4 * (g.n + 1) + 12 * g.m + S * (4 * g.m + 12 * g.n) + 4 * S
        gbs = (nb_f + nb_b) / ((fm + bm) * 1e-3) / 1e9
        resident = (4 * g.m * S + 8 * g.n * S) / 1e9
        print(f"{S:5d} {fm:8.3f} {bm:8.3f} {pm:9.3f} {gbs:12.0f} {gbs / peak:6.2f} "
              f"{2 * g.m * S / ((fm + bm) * 1e-3):15.3e} {resident:12.1f}", flush=True)
        del D
    G.close()


if __name__ == "__main__":
    main()
