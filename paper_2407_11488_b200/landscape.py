"""Reporting over tuning caches: tuning impact and top-k.

Only the consumers the hot path reports through:
``perf_stats`` follows ref `pkg/src/tunescape/landscape.py:85-102`
(impact = max perf / median perf over ok records, perf = stored metric
or ``1/time_ms``, ``statistics.median``) and adds the north_star's
best/worst ratio; ``top_k`` follows ref :453-461 (ties broken on the
string key).  Fitness-flow graphs, PageRank and portability stay in the
reference (out of scope): caches written here import
there unchanged.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass

from .errors import NoFeasibleData
from .measure import Observation


def metric_of(o: Observation) -> float:
    return o.metric_value if o.metric_value is not None else 1.0 / o.time_ms


@dataclass(frozen=True)
class PerfStats:
    n_ok: int
    n_failed: int
    median_perf: float
    max_perf: float
    min_time_ms: float
    impact: float  # max_perf / median_perf (paper's "tuning impact")
    min_perf: float = 0.0
    best_over_worst: float = 0.0  # max_perf / min_perf (north_star addition)


def perf_stats(cache) -> PerfStats:
    ok = cache.ok_records()
    if not ok:
        raise NoFeasibleData(f"cache {cache.kernel_name}/{cache.device_name} has no successful records")
    perfs = [metric_of(o) for o in ok.values()]
    med = statistics.median(perfs)
    hi, lo = max(perfs), min(perfs)
    return PerfStats(n_ok=len(ok), n_failed=cache.n_failed(), median_perf=med, max_perf=hi,
                     min_time_ms=min(o.time_ms for o in ok.values()), impact=hi / med,
                     min_perf=lo, best_over_worst=hi / lo)


def top_k(cache, k: int = 5) -> list:
    """The k best ok records as (key, perf), ties broken by key string."""
    ok = cache.ok_records()
    ranked = sorted(ok.items(), key=lambda kv: (-metric_of(kv[1]), kv[0]))
    return [(key, metric_of(o)) for key, o in ranked[:k]]
