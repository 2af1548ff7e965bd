"""bench.py multi-rank plumbing on the CPU (gloo): `bench.py --gpus N` spawns N
ranks itself (torch.distributed.run) when it is not already under torchrun,
shards the envs contiguously, and seeds every env from SeedSequence([seed,
env]) so the workload does not depend on N."""

import json
import subprocess
import sys

from conftest import ROOT


def _run(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_dry_run_two_ranks_matches_one():
    one = _run("--gpus", "1", "--dry-run", "--envs", "16")
    two = _run("--gpus", "2", "--dry-run", "--envs", "16")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["shards"] == [[0, 8], [8, 16]]
    assert one["shards"] == [[0, 16]]
    # the same per-env inputs whatever the rank count
    assert abs(one["input_checksum"] - two["input_checksum"]) < 1e-6 * abs(one["input_checksum"]) + 1e-9
    assert one["sign_counts"] == two["sign_counts"] == [8, 0, 8]
    assert two["max_over_ranks"] == 2.0


def test_env_inputs_are_shard_independent():
    sys.path.insert(0, str(ROOT))
    import numpy as np

    import bench

    a = bench.shard_inputs(0, 6)
    b = [np.concatenate([x, y]) for x, y in zip(bench.shard_inputs(0, 3), bench.shard_inputs(3, 6))]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
