"""Footprint KPIs — TEST/BENCH INFRASTRUCTURE (part of the oracle).

PAPER.md:26 (§Sustainability measures):
    %RAM       = (dataRAM + bufferRAM) / dataRAM
    tFootprint = avg(%RAM) * runTime
(eFootprint = avg(%RAM) * Energy is out of scope: no RAPL on the GPU box.)

Reading R6: the buffer lives for the whole call, so avg(%RAM) is
its peak.  Pinned in tests/test_footprint.py by the paper's Table Squidtab
(PAPER.md:481-497): r(pcdF) = r(%M) * r(pcdE) for every column within the
table's 2-decimal rounding, and by the SPEC.md:419-430 examples.
"""
from __future__ import annotations


def ram_pct(data_bytes: float, buffer_bytes: float) -> float:
    if data_bytes <= 0:
        raise ValueError("dataRAM must be > 0")
    return (data_bytes + buffer_bytes) / data_bytes


def t_footprint(avg_ram_pct: float, run_time: float) -> float:
    if run_time < 0:
        raise ValueError("runTime must be >= 0")
    return avg_ram_pct * run_time


def ratio(numerator: float, denominator: float) -> float:
    """Squidtab-style ratio of two algorithms' KPI medians."""
    return numerator / denominator
