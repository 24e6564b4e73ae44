"""Scenario sharding for the multi-GPU batch path (host logic, no CUDA).

Batched what-if scenarios are independent (timing views), so
they shard across ranks with no data-path collective: rank r owns a contiguous
block of scenario ids -- the equal-load special case of the paper's balanced
bin packing of GPU work.  The only collective is the final
all-gather of each rank's worst slacks (BASELINE.json:5), done by hf_run_batch
through NCCL; rank r's block lands at offset r * s_local of wns_all.
"""
from __future__ import annotations


def scenario_block(rank: int, world: int, scenarios: int, scaling: str = "weak"):
    """[begin, end) of the global scenario ids owned by `rank`.

    weak:   every rank owns `scenarios` ids (rank r: [r*S, (r+1)*S)).
    strong: `scenarios` ids in total, split as evenly as possible (C4: 64 over G).
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if scaling == "weak":
        return rank * scenarios, (rank + 1) * scenarios
    if scaling == "strong":
        return rank * scenarios // world, (rank + 1) * scenarios // world
    raise ValueError(scaling)


def gather_layout(blocks):
    """Offsets of each rank's block in the gathered array (all blocks equal size,
    as NCCL all-gather requires); raises if the blocks are ragged."""
    sizes = {e - b for b, e in blocks}
    if len(sizes) != 1:
        raise ValueError("all-gather needs equal scenario blocks per rank")
    s = sizes.pop()
    return [r * s for r in range(len(blocks))]
