"""Batch sharding of independent deblurring problems across ranks.

The batched configuration (BASELINE.json configs[3]: 64 independent 1024^2
problems, PSFs alternating Gaussian / box) shards with no collective on the
hot path: every rank solves its own problems and only the timing / report
reduction crosses ranks.  Problems are dealt round-robin in pairs so every
rank gets the same mix of Gaussian (even index) and box (odd index) PSFs,
which balances the per-rank PCG iteration totals (box problems need ~29%
more iterations).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_problems(num_problems: int, world: int, rank: int) -> list[int]:
    """Problem indices owned by ``rank``: pairs (2k, 2k+1) dealt round-robin."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    pairs = [list(range(i, min(i + 2, num_problems))) for i in range(0, num_problems, 2)]
    mine: list[int] = []
    for k, pair in enumerate(pairs):
        if k % world == rank:
            mine.extend(pair)
    return mine


def reduce_run(elapsed_s: float, iterations: int, launches: int = 0,
               device: torch.device | None = None) -> tuple[float, int, int]:
    """Max elapsed over ranks and summed work counters (identity without a process group)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return elapsed_s, iterations, launches
    dev = device or torch.device("cpu")
    t = torch.tensor([elapsed_s], dtype=torch.float64, device=dev)
    c = torch.tensor([float(iterations), float(launches)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t[0]), int(c[0]), int(c[1])
