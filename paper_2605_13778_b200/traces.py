"""Round-trace wire format: ``RoundRecord`` JSONL, byte-compatible with the
reference so ``specflow report`` (bench/reports.py, bench/metrics.py) can
re-aggregate runs of the B200 path.

Mirrors:
  * ``RoundRecord`` / ``to_record``          runtime.py:91-129
  * ``dump_json_line`` / ``write_trace`` /
    ``read_trace``                           bench/reports.py:96-114
  * ``episode_stats``                        bench/metrics.py:45-75

``records_from_device`` turns the device decision words of a batched flash
round (``ActionExpert.flash_batch`` / ``sf_ae_flash_round``: prefix L, switch,
path code, planned) into per-env records, so batched GPU runs produce the same
trace schema as the reference's sequential episode loop.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Mapping, Sequence

import numpy as np

from ._capi import (SF_PATH_FLASH_ACCEPTED, SF_PATH_FLASH_PHASE, SF_PATH_FLASH_REJECTED,
                    SF_RES_PATH, SF_RES_PLANNED, SF_RES_PREFIX, SF_RES_SWITCH)
from .runtime import (PATH_FLASH_ACCEPTED, PATH_FLASH_PHASE, PATH_FLASH_REJECTED, PATH_FULL,
                      PATH_PERIODIC)

_DEVICE_PATH = {
    SF_PATH_FLASH_ACCEPTED: PATH_FLASH_ACCEPTED,
    SF_PATH_FLASH_REJECTED: PATH_FLASH_REJECTED,
    SF_PATH_FLASH_PHASE: PATH_FLASH_PHASE,
}


@dataclass
class RoundRecord:
    """One replanning round (runtime.py:91-109)."""

    index: int
    path: str
    executed: int
    latency_ms: float
    start_tick: int
    stall_ticks: int
    planned: int
    prefix: int | None = None
    branch_prefixes: tuple[int, ...] | None = None
    gripper_switch: bool | None = None
    switch_in_executed: bool | None = None
    cache_round: int | None = None
    denoise_seed: int | None = None
    verify_seed: int | None = None
    terminal: str | None = None

    def to_record(self, **extra) -> dict:
        """Same keys and value types as runtime.py:111-129."""
        rec = {
            "round": self.index,
            "path": self.path,
            "executed": self.executed,
            "latency_ms": self.latency_ms,
            "start_tick": self.start_tick,
            "stall_ticks": self.stall_ticks,
            "planned": self.planned,
            "prefix": self.prefix,
            "branch_prefixes": list(self.branch_prefixes) if self.branch_prefixes is not None else None,
            "gripper_switch": self.gripper_switch,
            "switch_in_executed": self.switch_in_executed,
            "cache_round": self.cache_round,
            "denoise_seed": self.denoise_seed,
            "verify_seed": self.verify_seed,
            "terminal": self.terminal,
        }
        rec.update(extra)
        return rec


def dump_json_line(record: Mapping) -> str:
    """reports.py:96-97: sorted keys, compact separators."""
    return json.dumps(record, sort_keys=True, separators=(",", ":"))


def write_trace(path: str | Path, records: Iterable[Mapping]) -> None:
    """reports.py:100-104: one JSON object per line."""
    with open(path, "w", encoding="utf-8") as fh:
        for rec in records:
            fh.write(dump_json_line(rec))
            fh.write("\n")


def read_trace(path: str | Path) -> list[dict]:
    """reports.py:107-114."""
    records = []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if line:
                records.append(json.loads(line))
    return records


@dataclass(frozen=True)
class EpisodeStats:
    success: bool
    rounds: int
    flash_rounds: int
    flash_rate: float
    acc: float
    lat_ms: float
    per_action_ms: float
    total_latency_ms: float
    executed_actions: int
    speedup: float


def episode_stats(records: Sequence[Mapping], success: bool, replan_size: int,
                  baseline_full_ms: float) -> EpisodeStats:
    """Fold round records into episode metrics (metrics.py:45-75)."""
    if not records:
        raise ValueError("episode trace is empty")
    rounds = len(records)
    flash_accepted = [r for r in records if r["path"] == PATH_FLASH_ACCEPTED]
    total_latency = float(sum(r["latency_ms"] for r in records))
    executed = int(sum(r["executed"] for r in records))
    lat = total_latency / rounds
    acc = (sum(r["executed"] for r in flash_accepted) / (replan_size * len(flash_accepted))
           if flash_accepted else 0.0)
    return EpisodeStats(success=success, rounds=rounds, flash_rounds=len(flash_accepted),
                        flash_rate=len(flash_accepted) / rounds, acc=acc, lat_ms=lat,
                        per_action_ms=total_latency / executed if executed else float("nan"),
                        total_latency_ms=total_latency, executed_actions=executed,
                        speedup=baseline_full_ms / lat if lat > 0 else float("nan"))


def records_from_device(result: np.ndarray, branch: np.ndarray | None, round_index: int,
                        latency_ms: float, start_ticks: Sequence[int] | None = None,
                        verify_seeds: Sequence[int] | None = None,
                        cache_rounds: Sequence[int] | None = None) -> list[RoundRecord]:
    """Per-env records of one batched flash round from the device decision
    words ``result [B, 8]`` (and branch prefixes ``[B, K]``). ``executed`` is
    the planned prefix (the conveyor stepping that would clip it is out of
    scope); fallback rounds carry the path label and ``planned = replan_size``
    as the reference does before its full round (runtime.py:289-309)."""
    result = np.asarray(result)
    recs = []
    for e in range(result.shape[0]):
        w = result[e]
        path = _DEVICE_PATH.get(int(w[SF_RES_PATH]))
        if path is None:
            raise ValueError(f"env {e}: unknown device path code {int(w[SF_RES_PATH])}")
        planned = int(w[SF_RES_PLANNED])
        recs.append(RoundRecord(
            index=round_index, path=path, executed=planned if path == PATH_FLASH_ACCEPTED else 0,
            latency_ms=float(latency_ms), start_tick=int(start_ticks[e]) if start_ticks is not None else 0,
            stall_ticks=0, planned=planned, prefix=int(w[SF_RES_PREFIX]),
            branch_prefixes=tuple(int(x) for x in branch[e]) if branch is not None else None,
            gripper_switch=bool(w[SF_RES_SWITCH]),
            cache_round=int(cache_rounds[e]) if cache_rounds is not None else None,
            verify_seed=int(verify_seeds[e]) if verify_seeds is not None else None))
    return recs


__all__ = ["RoundRecord", "dump_json_line", "write_trace", "read_trace", "EpisodeStats",
           "episode_stats", "records_from_device", "PATH_FULL", "PATH_PERIODIC"]
