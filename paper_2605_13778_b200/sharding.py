"""Environment sharding across GPUs.

Environments are independent (per-env runner state, seeds and prefix KV,
runtime.py:133-139, harness.py:435-436), so the batched path shards them
contiguously across ranks with NO collective on the hot path. The only
communication is after the timed region: a max-over-ranks reduction of the
device time and an all-gather of per-rank decision counters.
"""

from __future__ import annotations

import numpy as np
import torch


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) env block of `rank`; remainders go to the first ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def env_seed(episode_seed: int, env: int) -> int:
    """Per-env stream seed: SeedSequence([seed, env]) like harness.py:435-436."""
    return int(np.random.SeedSequence([int(episode_seed), int(env)]).generate_state(1)[0])


def max_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_counts(counts: torch.Tensor) -> torch.Tensor:
    """All-gather per-rank decision counters ([3] = accepted/rejected/phase)
    after the timed region; returns the element-wise sum over ranks."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return counts.clone()
    out = [torch.empty_like(counts) for _ in range(dist.get_world_size())]
    dist.all_gather(out, counts)
    return torch.stack(out).sum(0)


def decision_counts(result: torch.Tensor) -> torch.Tensor:
    """Histogram of SF_RES_PATH over envs from the device result words."""
    return torch.bincount(result[:, 2].long(), minlength=3)[:3]
