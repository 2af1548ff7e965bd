"""Round-trace wire format: ``RoundRecord`` JSONL, byte-compatible with the
reference so ``specflow report`` (bench/reports.py, bench/metrics.py) can
re-aggregate runs of the B200 path.

Mirrors:
  * ``RoundRecord`` / ``to_record``          runtime.py:91-129
  * ``dump_json_line`` / ``write_trace`` /
    ``read_trace``                           bench/reports.py:96-114
  * ``episode_stats``                        bench/metrics.py:45-75

``records_from_device`` turns a batched replanning round
(``BatchedReplanner.round``: post-bookkeeping path codes and planned prefixes,
plus the flash attempt's prefix / branch / switch words) into per-env records, so batched GPU runs produce the same
trace schema as the reference's sequential episode loop.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Mapping, Sequence

import numpy as np

from ._capi import (SF_PATH_FLASH_ACCEPTED, SF_PATH_FLASH_PHASE, SF_PATH_FLASH_REJECTED,
                    SF_PATH_FULL, SF_PATH_PERIODIC, SF_RES_PREFIX, SF_RES_SWITCH)
from .runtime import (PATH_FLASH_ACCEPTED, PATH_FLASH_PHASE, PATH_FLASH_REJECTED, PATH_FULL,
                      PATH_PERIODIC)

_DEVICE_PATH = {
    SF_PATH_FLASH_ACCEPTED: PATH_FLASH_ACCEPTED,
    SF_PATH_FLASH_REJECTED: PATH_FLASH_REJECTED,
    SF_PATH_FLASH_PHASE: PATH_FLASH_PHASE,
    SF_PATH_FULL: PATH_FULL,
    SF_PATH_PERIODIC: PATH_PERIODIC,
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


def records_from_device(path: np.ndarray, planned: np.ndarray, result: np.ndarray,
                        branch: np.ndarray | None, round_index: int, latency_ms: float,
                        start_ticks: Sequence[int] | None = None,
                        verify_seeds: Sequence[int] | None = None,
                        cache_rounds: Sequence[int] | None = None,
                        switch_in_executed: np.ndarray | None = None) -> list[RoundRecord]:
    """Per-env records of one batched replanning round.

    ``path`` / ``planned`` [B] are the round's POST-bookkeeping values
    (``BatchedReplanner.round``: ``sf_replan_update``), so full rounds (no
    context yet) and periodic refreshes get their own labels and planned =
    replan_size, exactly as ``run_episode`` records them (runtime.py:262-276).
    ``result [B, 8]`` / ``branch [B, K]`` are the flash attempt's decision
    words; as in the reference they are recorded only for rounds that made a
    flash attempt (accepted and both fallbacks, runtime.py:279-282).
    ``executed`` = planned for every path (the conveyor stepping that could
    clip it at episode end is out of scope; runtime.py:325-326).
    ``switch_in_executed`` [B] (optional, ``BatchedReplanner``'s device
    flag) is recorded for accepted rounds only (runtime.py:321-323)."""
    path, planned, result = np.asarray(path), np.asarray(planned), np.asarray(result)
    recs = []
    for e in range(path.shape[0]):
        code = int(path[e])
        label = _DEVICE_PATH.get(code)
        if label is None:
            raise ValueError(f"env {e}: unknown device path code {code}")
        flash = code in (SF_PATH_FLASH_ACCEPTED, SF_PATH_FLASH_REJECTED, SF_PATH_FLASH_PHASE)
        w = result[e]
        sie = None
        if code == SF_PATH_FLASH_ACCEPTED and switch_in_executed is not None:
            sie = bool(switch_in_executed[e])
        recs.append(RoundRecord(
            index=round_index, path=label, executed=int(planned[e]), latency_ms=float(latency_ms),
            start_tick=int(start_ticks[e]) if start_ticks is not None else 0, stall_ticks=0,
            planned=int(planned[e]),
            prefix=int(w[SF_RES_PREFIX]) if flash else None,
            branch_prefixes=(tuple(int(x) for x in branch[e]) if flash and branch is not None
                             else None),
            gripper_switch=bool(w[SF_RES_SWITCH]) if flash else None,
            switch_in_executed=sie,
            cache_round=int(cache_rounds[e]) if flash and cache_rounds is not None else None,
            verify_seed=int(verify_seeds[e]) if flash and verify_seeds is not None else None))
    return recs


__all__ = ["RoundRecord", "dump_json_line", "write_trace", "read_trace", "EpisodeStats",
           "episode_stats", "records_from_device", "PATH_FULL", "PATH_PERIODIC"]
