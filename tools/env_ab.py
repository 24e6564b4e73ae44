"""A/B timing of library settings read from the environment at call time, on one
graph in one process: every variant runs `--reps` times, interleaved.

    python tools/env_ab.py --config C5 --S 1 [--single] --var HF_W1_NU=1 --var HF_W1_NU=2,HF_W1_DBG=1

Prints per variant the median forward / backward kernel ms (CUDA events inside the
library, L2 flushed before each call) and the f+b GB/s of the algorithmic bytes.
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
    ap.add_argument("--config", default="C5")
    ap.add_argument("--S", type=int, default=1)
    ap.add_argument("--graph", default=None, help="graph of another config (e.g. C3 for C4)")
    ap.add_argument("--single", action="store_true", help="single-graph calls (graph delays, S=1)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--var", action="append", default=[])
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = hfgen.config(a.config)
    st = torch.cuda.current_stream()
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev),
                           delay=torch.from_numpy(g.delay).to(dev), stream=st)
    hf.hf_profile_enable(G, True)
    L = hf.hf_levelize(G)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    at_src = torch.from_numpy(g.at_src).to(dev)
    S = 1 if a.single else a.S
    at = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    rat = torch.empty(g.n * S, dtype=torch.float32, device=dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    D = None if a.single else torch.from_numpy(hfgen.scenario_delays(g, 0, S, "ms")).to(dev)
    T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
    nb_f = 4 * (g.n + 1) + 8 * g.m + S * (4 * g.m + 8 * g.n)
    nb_b = 4 * (g.n + 1) + 12 * g.m + S * (4 * g.m + 12 * g.n) + 4 * S
    variants = a.var or [""]
    res = {v: ([], [], []) for v in variants}
    base_env = dict(os.environ)
    print(f"{a.config}: n={g.n} m={g.m} L={L} S={S} {'single' if a.single else 'batch'}")
    for r in range(a.reps + 1):
        for v in variants:
            os.environ.clear()
            os.environ.update(base_env)
            for kv in filter(None, v.split(",")):
                k, val = kv.split("=")
                os.environ[k] = val
            flush.fill_(1.0)
            if a.single:
                hf.hf_propagate_forward(G, at_src, at)
                hf.hf_propagate_backward(G, float(g.t_req), at, rat, None, w)
            else:
                hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w, at=at, rat=rat)
            _, fm, bm, _ = hf.hf_profile_read(G)
            ph = hf.hf_profile_read_batch(G) if not a.single else fm + bm
            if r:
                res[v][0].append(fm)
                res[v][1].append(bm)
                res[v][2].append(ph)
    os.environ.clear()
    os.environ.update(base_env)
    for v in variants:
        fm, bm = float(np.median(res[v][0])), float(np.median(res[v][1]))
        ph = float(np.median(res[v][2]))
        print(f"{v or '(default)':40s} fwd {fm:7.3f} ms  bwd {bm:7.3f} ms  f+b {fm + bm:7.3f} ms "
              f"{(nb_f + nb_b) / (fm + bm) / 1e6:7.1f} GB/s  phase {ph:7.3f} ms "
              f"({(nb_f + nb_b) / ph / 1e6:7.1f} GB/s)")


if __name__ == "__main__":
    main()
