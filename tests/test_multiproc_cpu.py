"""Multi-process (gloo, world_size 2) checks of the env-sharding plumbing used
by bench.py under torchrun: shards partition the envs, per-env seeds are
rank-independent, the max-over-ranks timing and the decision-counter gather
are the only collectives and give the same answer on every rank."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_13778_b200.sharding import (decision_counts, env_seed, gather_counts,
                                                max_over_ranks, shard_range)

    lo, hi = shard_range(total, rank, world)
    seeds = [env_seed(7, e) for e in range(lo, hi)]
    t = max_over_ranks(10.0 + rank)
    # fake device result words: path code = env % 3
    res = torch.zeros((hi - lo, 8), dtype=torch.int32)
    res[:, 2] = torch.arange(lo, hi) % 3
    counts = gather_counts(decision_counts(res))
    q.put((rank, lo, hi, seeds, t, counts.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [512, 13])
def test_two_rank_sharding(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2605_13778_b200.sharding import env_seed

    covered = []
    for rank, lo, hi, seeds, t, counts in out:
        covered += list(range(lo, hi))
        assert seeds == [env_seed(7, e) for e in range(lo, hi)]
        assert t == 11.0  # max over ranks, identical everywhere
        want = torch.bincount(torch.arange(total) % 3, minlength=3).tolist()
        assert counts == want
    assert covered == list(range(total))


def test_shard_range_edges():
    from paper_2605_13778_b200.sharding import shard_range

    for total in (0, 1, 7, 512):
        for world in (1, 2, 3, 8):
            blocks = [shard_range(total, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
