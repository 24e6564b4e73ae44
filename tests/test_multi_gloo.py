"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded batch path:
scenario blocks partition the global scenario ids, and per-rank worst slacks
all-gathered in rank order equal the unsharded result bit for bit (SURVEY.md
§8(e), P9 shard invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hfgen
import oracle
from paper_2203_08395_b200.shard import gather_layout, scenario_block


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, S_per_rank, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g = hfgen.config("C1", 0.5)
    lo, hi = scenario_block(rank, world, S_per_rank, "weak")
    D = hfgen.scenario_delays(g, lo, hi, "ms")
    T = np.full(hi - lo, g.t_req, np.float32)
    w = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=1)
    t = torch.from_numpy(w.copy())
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    if rank == 0:
        np.save(out_path, torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_scenario_blocks_partition():
    for world in (1, 2, 4, 8):
        for scaling, S in (("weak", 64), ("strong", 64)):
            blocks = [scenario_block(r, world, S, scaling) for r in range(world)]
            ids = np.concatenate([np.arange(b, e) for b, e in blocks])
            total = S * world if scaling == "weak" else S
            assert np.array_equal(ids, np.arange(total))
            assert gather_layout(blocks) == [r * (total // world) for r in range(world)]
    with pytest.raises(ValueError):
        gather_layout([(0, 3), (3, 5)])


def test_two_rank_gather_equals_unsharded(tmp_path):
    world, S = 2, 3
    port = _free_port()
    out = str(tmp_path / "wns_all.npy")
    mp.start_processes(_worker, args=(world, port, S, out), nprocs=world, join=True,
                       start_method="spawn")
    gathered = np.load(out)
    g = hfgen.config("C1", 0.5)
    D = hfgen.scenario_delays(g, 0, world * S, "ms")
    T = np.full(world * S, g.t_req, np.float32)
    full = oracle.batch(g.n, g.m, g.in_ptr, g.in_src, D, T, g.at_src, "ms", threads=2)
    assert np.array_equal(gathered.view(np.uint32), full.view(np.uint32))
