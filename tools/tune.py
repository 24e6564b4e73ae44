"""Propagation tuning sweep: one graph, many HF_* settings (read per call by libhf).

    python tools/tune.py --config C3 --S 64 --grid 'HF_RB=4,8;HF_POLL_ALL=0,1'
"""
import argparse
import itertools
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
    ap.add_argument("--S", type=int, default=64)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--grid", default="")
    ap.add_argument("--sets", default="", help="explicit settings separated by '|'")
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
    S = a.S
    D = torch.from_numpy(hfgen.scenario_delays(g, 0, S, "ms")).to(dev)
    T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    settings = []
    if a.grid:
        keys, vals = [], []
        for part in a.grid.split(";"):
            k, v = part.split("=")
            keys.append(k)
            vals.append(v.split(","))
        for combo in itertools.product(*vals):
            settings.append(dict(zip(keys, combo)))
    for s in a.sets.split("|") if a.sets else []:
        settings.append(dict(kv.split("=") for kv in s.split()) if s.strip() else {})
    if not settings:
        settings = [{}]
    nb_f = 4 * (g.n + 1) + 8 * g.m + S * (4 * g.m + 8 * g.n)
    nb_b = 4 * (g.n + 1) + 12 * g.m + S * (4 * g.m + 12 * g.n) + 4 * S
    ref = None
    print(f"{a.config}: n={g.n} m={g.m} L={L} S={S}")
    for cfg in settings:
        for k in [k for k in os.environ if k.startswith("HF_")]:
            if k not in ("HF_NCCL_LIBRARY",):
                del os.environ[k]
        os.environ.update(cfg)
        f, b, pp = [], [], []
        for r in range(a.reps + 1):
            flush.fill_(1.0)
            hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, at_src, w)
            _, fm, bm, _ = hf.hf_profile_read(G)
            ph = hf.hf_profile_read_batch(G)
            if r > 0:
                f.append(fm)
                b.append(bm)
                pp.append(ph)
        res = w.cpu().numpy().view(np.uint32).copy()
        same = "" if ref is None else ("" if np.array_equal(ref, res) else "  WNS MISMATCH")
        ref = res if ref is None else ref
        fm, bm, pm = float(np.median(f)), float(np.median(b)), float(np.median(pp))
        print(f"{' '.join(f'{k}={v}' for k, v in cfg.items()):40s} fwd {fm:7.3f} ms "
              f"bwd {bm:7.3f} ms  phase {pm:7.3f} ms ({(nb_f + nb_b) / pm / 1e6:6.0f} GB/s)"
              f"{same}", flush=True)


if __name__ == "__main__":
    main()
