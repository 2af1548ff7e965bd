"""RoundRecord JSONL wire format (traces.py) against fixtures written by the
reference itself (tests/golden/make_trace_golden.py): byte-identical traces,
identical episode statistics, and device decision words -> records."""

import dataclasses
import json
from pathlib import Path

import numpy as np

from paper_2605_13778_b200 import traces
from paper_2605_13778_b200._capi import (SF_PATH_FLASH_ACCEPTED, SF_PATH_FLASH_PHASE,
                                         SF_PATH_FLASH_REJECTED)

GOLD = Path(__file__).resolve().parent / "golden"


def _records():
    rows = json.loads((GOLD / "trace_ref_records.json").read_text())
    out = []
    for r in rows:
        if r.get("branch_prefixes") is not None:
            r["branch_prefixes"] = tuple(r["branch_prefixes"])
        out.append(traces.RoundRecord(**r))
    return out


def test_trace_bytes_match_reference(tmp_path):
    recs = [r.to_record(episode_seed=7, speed=0.12, variant="flash") for r in _records()]
    p = tmp_path / "t.jsonl"
    traces.write_trace(p, recs)
    assert p.read_bytes() == (GOLD / "trace_ref.jsonl").read_bytes()
    assert traces.read_trace(p) == traces.read_trace(GOLD / "trace_ref.jsonl")


def test_episode_stats_match_reference():
    recs = [r.to_record() for r in _records()]
    got = dataclasses.asdict(traces.episode_stats(recs, True, 12, 58.0))
    want = json.loads((GOLD / "trace_ref_stats.json").read_text())
    assert got.keys() == want.keys()
    for k in want:
        assert got[k] == want[k], k


def test_records_from_device_words():
    """Batched replanner round -> records: full / periodic rounds keep their
    labels and carry no flash fields; fallbacks execute replan_size actions
    (runtime.py:262-326)."""
    from paper_2605_13778_b200._capi import SF_PATH_FULL, SF_PATH_PERIODIC

    result = np.zeros((5, 8), dtype=np.int32)
    result[0, :4] = [7, 0, SF_PATH_FLASH_ACCEPTED, 7]
    result[1, :4] = [0, 0, SF_PATH_FLASH_REJECTED, 12]
    result[2, :4] = [5, 1, SF_PATH_FLASH_PHASE, 12]
    result[3, :4] = [9, 0, SF_PATH_FLASH_ACCEPTED, 9]   # attempt never used (no context yet)
    result[4, :4] = [3, 0, SF_PATH_FLASH_ACCEPTED, 3]   # attempt never used (periodic refresh)
    path = np.array([SF_PATH_FLASH_ACCEPTED, SF_PATH_FLASH_REJECTED, SF_PATH_FLASH_PHASE,
                     SF_PATH_FULL, SF_PATH_PERIODIC])
    planned = np.array([7, 12, 12, 12, 12])
    branch = np.array([[9, 7], [0, 3], [5, 6], [9, 9], [3, 4]])
    recs = traces.records_from_device(path, planned, result, branch, round_index=4, latency_ms=1.1,
                                      verify_seeds=[11, 12, 13, 14, 15], cache_rounds=[0, 0, 2, 0, 0],
                                      switch_in_executed=np.array([1, 0, 0, 0, 0]))
    assert [r.path for r in recs] == ["flash_accepted", "flash_rejected_fallback", "flash_phase_fallback",
                                      "full", "periodic_refresh"]
    assert [r.planned for r in recs] == [7, 12, 12, 12, 12]
    assert [r.executed for r in recs] == [7, 12, 12, 12, 12]
    assert recs[0].branch_prefixes == (9, 7) and recs[2].gripper_switch is True
    assert recs[0].switch_in_executed is True and recs[1].switch_in_executed is None
    for r in recs[3:]:
        assert r.prefix is None and r.branch_prefixes is None and r.gripper_switch is None
        assert r.verify_seed is None and r.cache_round is None
    line = traces.dump_json_line(recs[0].to_record())
    assert json.loads(line)["path"] == "flash_accepted"
