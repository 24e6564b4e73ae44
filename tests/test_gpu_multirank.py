"""Two ranks through libhf: the strong-scaling split of C4 (the
scenarios of one batch divided over the ranks, BASELINE.json:10) run as two
processes, each creating its own graph and running hf_run_batch_d on its scenario
block, the per-rank worst slacks all-gathered (torch.distributed, gloo) in rank
order -- bit-identical to the oracle over all scenarios.

Both ranks use cuda:0 (the box has one GPU); their kernels never wait on each other
(independent shards, the gather is on the host), so this is the multi-rank data path
of the product minus the NCCL transport, whose single-rank form is
test_batch_nccl_gather_single_rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hfgen
import oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, scale, S_total, out_path):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2203_08395_b200 import hf
    from paper_2203_08395_b200.shard import scenario_block
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dev = torch.device("cuda:0")
    g = hfgen.config(cfg, scale)
    lo, hi = scenario_block(rank, world, S_total, "strong")
    S = hi - lo
    D = torch.from_numpy(hfgen.scenario_delays(g, lo, hi, "ms")).to(dev)
    T = torch.full((S,), g.t_req, dtype=torch.float32, device=dev)
    G = hf.hf_graph_create(g.n, g.m, torch.from_numpy(g.in_ptr).to(dev),
                           torch.from_numpy(g.in_src).to(dev),
                           delay=torch.from_numpy(g.delay).to(dev),
                           stream=torch.cuda.current_stream())
    hf.hf_levelize(G)
    w = torch.empty(S, dtype=torch.float32, device=dev)
    hf.hf_run_batch(G, S, D, hf.HF_LAYOUT_MS, T, torch.from_numpy(g.at_src).to(dev), w)
    hf.hf_sync(G)
    t = w.cpu()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    if rank == 0:
        np.save(out_path, torch.cat(parts).numpy())
    G.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,scale,S_total", [("C1", 1.0, 16), ("C3", 0.1, 128)])
def test_two_ranks_strong_split_bit_exact(tmp_path, cfg, scale, S_total):
    world = 2
    out = str(tmp_path / "wns_all.npy")
    mp.start_processes(_worker, args=(world, _free_port(), cfg, scale, S_total, out),
                       nprocs=world, join=True, start_method="spawn")
    gathered = np.load(out)
    g = hfgen.config(cfg, scale)
    D = hfgen.scenario_delays(g, 0, S_total, "ms")
    T = np.full(S_total, g.t_req, np.float32)
    full = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=8)
    assert np.array_equal(gathered.view(np.uint32), full.view(np.uint32))
