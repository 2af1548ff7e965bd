"""Golden fixture for the RoundRecord JSONL wire format (traces.py).

Run in the build container (the reference is importable read-only there):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_trace_golden.py
Writes trace_ref.jsonl (reference runtime.RoundRecord.to_record +
bench.reports.write_trace) and trace_ref_stats.json (bench.metrics.episode_stats).
"""

import dataclasses
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from specflow.bench.metrics import episode_stats  # noqa: E402
from specflow.bench.reports import write_trace  # noqa: E402
from specflow.runtime import RoundRecord  # noqa: E402

HERE = Path(__file__).resolve().parent

RECORDS = [
    dict(index=0, path="full", executed=12, latency_ms=58.0, start_tick=0, stall_ticks=3, planned=12,
         denoise_seed=123456789),
    dict(index=1, path="flash_accepted", executed=7, latency_ms=7.8, start_tick=15, stall_ticks=1,
         planned=7, prefix=7, branch_prefixes=(9, 7), gripper_switch=False, switch_in_executed=False,
         cache_round=0, verify_seed=987654321),
    dict(index=2, path="flash_rejected_fallback", executed=12, latency_ms=65.8, start_tick=23,
         stall_ticks=4, planned=12, prefix=0, branch_prefixes=(0, 3), gripper_switch=False,
         cache_round=0, denoise_seed=1, verify_seed=2),
    dict(index=3, path="flash_phase_fallback", executed=12, latency_ms=65.8, start_tick=39,
         stall_ticks=4, planned=12, prefix=5, branch_prefixes=(5, 6), gripper_switch=True,
         cache_round=2, denoise_seed=3, verify_seed=4),
    dict(index=4, path="periodic_refresh", executed=2, latency_ms=58.0, start_tick=55, stall_ticks=3,
         planned=12, denoise_seed=5, terminal="success"),
]


def main():
    recs = [RoundRecord(**r) for r in RECORDS]
    dicts = [r.to_record(episode_seed=7, speed=0.12, variant="flash") for r in recs]
    write_trace(HERE / "trace_ref.jsonl", dicts)
    stats = episode_stats([r.to_record() for r in recs], True, 12, 58.0)
    (HERE / "trace_ref_stats.json").write_text(json.dumps(dataclasses.asdict(stats), sort_keys=True))
    (HERE / "trace_ref_records.json").write_text(json.dumps(RECORDS, sort_keys=True))


if __name__ == "__main__":
    main()
