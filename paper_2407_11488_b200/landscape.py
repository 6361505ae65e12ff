"""Landscape analysis of tuning caches (SPEC.md ``landscape``).

The paper's three metric families, computed from a cache -- whether the
cache came from a B200 sweep here or from the paper's artifacts:

* **tuning impact** (:func:`perf_stats`): max performance / median
  performance over the ok records (perf = stored metric, else
  ``1/time_ms``), plus the north_star's best/worst ratio;
* **difficulty** (:func:`build_ffg`, :func:`pagerank`,
  :func:`proportion_of_centrality`, :func:`centrality_curve`): the fitness
  flow graph has an edge u -> v when v is a neighbour of u with a
  strictly smaller time; its sinks are the local minima, and C_p is the
  share of PageRank mass (damping 0.85, uniform teleport, dangling mass
  spread uniformly) held by minima within (1+p) of the optimum;
* **portability** (:func:`app_efficiency`, :func:`harmonic_pp`,
  :func:`perf_portability`, :func:`best_portable_config`): Eq. 2-3.

Plus the paper's tables and plot data: :func:`top_k`,
:func:`export_distribution`, :func:`export_dot`.

Design: everything graph-shaped is array code.  The flow graph is built
without materialising neighbour tuples -- a space is a mixed-radix number
system (``paramspace``), so a neighbour of node u is u's flat index plus
``(new - old) * stride`` of one parameter, and membership is one
``searchsorted`` over the ok nodes' flat indices.  The 116,928-node GEMM
space's graph builds in about a second (the reference's tuple loop takes
~8 s); PageRank is a ``bincount`` sparse mat-vec per power iteration.
"""

from __future__ import annotations

import json
import statistics
from dataclasses import dataclass, field
from pathlib import Path
from typing import Mapping, Sequence

import numpy as np

from .errors import (IncompleteCache, NoFeasibleData, NonConvergence, NoPortableConfiguration,
                     ProtocolError, UnknownDevice)
from .measure import Observation
from .paramspace import Config, NeighborScheme, config_key
from .store import TuningCache, check_space

DEFAULT_DAMPING = 0.85
DEFAULT_TOL = 1e-8
DEFAULT_MAX_ITER = 10_000


def p_grid(p_max: float = 0.15, step: float = 0.005) -> tuple:
    """Acceptable-optimum proportions 0, step, ..., p_max (rounded, inclusive)."""
    return tuple(round(i * step, 10) for i in range(int(round(p_max / step)) + 1))


DEFAULT_P_GRID = p_grid()  # 0% .. 15% in 0.5% steps (paper §6.1)
QUANTILE_PERCENTS = (1, 5, 25, 50, 75, 95, 99)


def metric_of(obs: Observation) -> float:
    """Performance of an ok observation: its metric, else ``1/time_ms``."""
    return obs.metric_value if obs.metric_value is not None else 1.0 / obs.time_ms


def _natural(key: str) -> tuple:
    """Sort key of a configuration key: integer fields compare as integers."""
    return tuple((0, int(f), "") if f.lstrip("-").isdigit() else (1, 0, f) for f in key.split(","))


def _no_data(cache: TuningCache) -> NoFeasibleData:
    return NoFeasibleData(f"cache {cache.kernel_name}/{cache.device_name} has no successful records")


# ---------------------------------------------------------------------------
# Tuning impact


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


def perf_stats(cache: TuningCache) -> PerfStats:
    ok = cache.ok_records()
    if not ok:
        raise _no_data(cache)
    perf = [metric_of(o) for o in ok.values()]
    mid, top, bottom = statistics.median(perf), max(perf), min(perf)
    return PerfStats(n_ok=len(ok), n_failed=cache.n_failed(), median_perf=mid, max_perf=top,
                     min_time_ms=min(o.time_ms for o in ok.values()), impact=top / mid,
                     min_perf=bottom, best_over_worst=top / bottom)


def top_k(cache: TuningCache, k: int = 5) -> list:
    """The k best ok records as ``(key, perf)``; ties in canonical order."""
    if k < 1:
        raise ProtocolError(f"top_k needs k >= 1, got {k}")
    ranked = sorted(cache.ok_records().items(), key=lambda kv: (-metric_of(kv[1]), _natural(kv[0])))
    return [(key, metric_of(o)) for key, o in ranked[:k]]


# ---------------------------------------------------------------------------
# Fitness flow graph


@dataclass
class FitnessFlowGraph:
    """Nodes = ok configurations (enumeration order); edges toward strictly faster neighbours."""

    scheme: NeighborScheme
    keys: tuple
    configs: tuple
    times: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    f_opt: float
    kernel_name: str = ""
    device_name: str = ""
    excluded_failures: int = 0
    _out_degrees: np.ndarray | None = field(default=None, repr=False)

    @property
    def n_nodes(self) -> int:
        return len(self.keys)

    @property
    def n_edges(self) -> int:
        return int(self.edge_src.size)

    @property
    def out_degrees(self) -> np.ndarray:
        if self._out_degrees is None:
            self._out_degrees = np.bincount(self.edge_src, minlength=self.n_nodes)
        return self._out_degrees

    def sinks(self) -> np.ndarray:
        return np.flatnonzero(self.out_degrees == 0)


def _neighbour_moves(space, scheme: NeighborScheme) -> list:
    """Per parameter: the position changes one move may make, as (param, old, new)."""
    moves = []
    for i, p in enumerate(space.parameters):
        n = len(p.values)
        for old in range(n):
            news = [j for j in range(n) if j != old] if scheme is NeighborScheme.HAMMING1 else \
                [j for j in (old - 1, old + 1) if 0 <= j < n]
            moves.extend((i, old, new) for new in news)
    return moves


def build_ffg(cache: TuningCache, space, scheme: NeighborScheme | str | None = None) -> FitnessFlowGraph:
    """The fitness flow graph of a *complete* cache over ``space``."""
    scheme = NeighborScheme(scheme) if scheme else space.neighbor_scheme
    check_space(cache, space)
    valid = space.valid_indices()
    configs_all = space.configs_at(valid)
    keys_all = [config_key(c) for c in configs_all]
    missing = sum(1 for k in keys_all if k not in cache.records)
    if missing:
        raise IncompleteCache(missing, len(keys_all))
    ok_mask = np.fromiter((cache.records[k].ok for k in keys_all), dtype=bool, count=len(keys_all))
    node_flat = valid[ok_mask]
    keys = tuple(k for k, m in zip(keys_all, ok_mask) if m)
    configs = tuple(c for c, m in zip(configs_all, ok_mask) if m)
    times = np.array([cache.records[k].time_ms for k in keys], dtype=np.float64)
    n = len(keys)
    src_parts, dst_parts, order_parts = [], [], []
    if n:
        strides = np.asarray(space.strides, dtype=np.int64)
        radices = np.asarray(space.radices, dtype=np.int64)
        digits = (node_flat[:, None] // strides[None, :]) % radices[None, :]
        nodes = np.arange(n, dtype=np.int64)
        for slot, (i, old, new) in enumerate(_neighbour_moves(space, scheme)):
            at = nodes[digits[:, i] == old]
            if at.size == 0:
                continue
            target = node_flat[at] + (new - old) * strides[i]
            pos = np.searchsorted(node_flat, target)
            hit = pos < n
            hit[hit] = node_flat[pos[hit]] == target[hit]
            u, v = at[hit], pos[hit]
            faster = times[v] < times[u]
            src_parts.append(u[faster])
            dst_parts.append(v[faster])
            # neighbour order of the reference: by parameter, then target position
            order_parts.append(np.full(int(faster.sum()), i * 4096 + new, dtype=np.int64))
    if src_parts:
        src, dst, rank = (np.concatenate(a) for a in (src_parts, dst_parts, order_parts))
        order = np.lexsort((rank, src))
        src, dst = src[order], dst[order]
    else:
        src = dst = np.zeros(0, dtype=np.int64)
    return FitnessFlowGraph(scheme=scheme, keys=keys, configs=configs, times=times, edge_src=src,
                            edge_dst=dst, f_opt=float(times.min()) if n else float("nan"),
                            kernel_name=cache.kernel_name, device_name=cache.device_name,
                            excluded_failures=int((~ok_mask).sum()))


def find_local_minima(g: FitnessFlowGraph) -> list:
    """Sinks of the graph (configurations without a faster neighbour)."""
    return [g.configs[i] for i in g.sinks()]


# ---------------------------------------------------------------------------
# PageRank and the proportion of centrality


def pagerank(g: FitnessFlowGraph, damping: float = DEFAULT_DAMPING, tol: float = DEFAULT_TOL,
             max_iter: int = DEFAULT_MAX_ITER) -> np.ndarray:
    """Power iteration: s' = d (P s + dangling(s)/n) + (1-d)/n until |s'-s|_1 < tol."""
    n = g.n_nodes
    if n == 0:
        raise NoFeasibleData("the flow graph has no nodes (every configuration failed)")
    deg = g.out_degrees.astype(np.float64)
    dangling = deg == 0
    inv_deg = np.where(dangling, 0.0, 1.0 / np.maximum(deg, 1.0))
    src, dst = g.edge_src, g.edge_dst
    s = np.full(n, 1.0 / n)
    residual = float("inf")
    for _ in range(max_iter):
        flow = np.bincount(dst, weights=(s * inv_deg)[src], minlength=n)
        nxt = damping * (flow + s[dangling].sum() / n) + (1.0 - damping) / n
        residual = float(np.abs(nxt - s).sum())
        s = nxt
        if residual < tol:
            return s
    raise NonConvergence(max_iter, residual, tol)


def proportion_of_centrality(g: FitnessFlowGraph, scores: np.ndarray, p: float) -> float:
    """C_p: centrality of minima within (1+p) of the optimum over that of all minima."""
    minima = g.sinks()
    weights = np.asarray(scores, dtype=np.float64)[minima]
    near = g.times[minima] <= (1.0 + p) * g.f_opt
    return float(weights[near].sum() / weights.sum())


@dataclass(frozen=True)
class CentralityCurve:
    p_grid: tuple
    c_p_values: tuple
    damping: float
    minima_count: int


def centrality_curve(g: FitnessFlowGraph, damping: float = DEFAULT_DAMPING,
                     p_grid: Sequence[float] | None = None, tol: float = DEFAULT_TOL,
                     max_iter: int = DEFAULT_MAX_ITER) -> CentralityCurve:
    grid = DEFAULT_P_GRID if p_grid is None else tuple(p_grid)
    scores = pagerank(g, damping, tol, max_iter)
    return CentralityCurve(grid, tuple(proportion_of_centrality(g, scores, p) for p in grid), damping,
                           int(g.sinks().size))


def write_centrality_csv(curve: CentralityCurve, path) -> Path:
    path = Path(path)
    rows = ["p,c_p"] + [f"{p!r},{c!r}" for p, c in zip(curve.p_grid, curve.c_p_values)]
    path.write_text("\n".join(rows) + "\n", encoding="utf-8")
    return path


write_curve_csv = write_centrality_csv


# ---------------------------------------------------------------------------
# Performance portability (Eq. 2-3)


@dataclass(frozen=True)
class PortabilityReport:
    devices: tuple
    config: str
    efficiencies: tuple
    pp: float

    def as_dict(self) -> dict:
        return {"devices": list(self.devices), "config": self.config,
                "efficiencies": list(self.efficiencies), "pp": self.pp}


def _key(config) -> str:
    return config if isinstance(config, str) else config_key(config)


def _best_perf(cache: TuningCache) -> float:
    ok = cache.ok_records()
    if not ok:
        raise _no_data(cache)
    return max(metric_of(o) for o in ok.values())


def app_efficiency(cache: TuningCache, config) -> float:
    """e_i = P_i(x) / max_x' P_i(x'); absent or failed configurations score 0."""
    obs = cache.records.get(_key(config))
    if obs is None or not obs.ok:
        return 0.0
    return metric_of(obs) / _best_perf(cache)


def harmonic_pp(efficiencies: Sequence[float]) -> float:
    """|H| / sum(1/e_i); any unsupported device (e_i = 0) gives 0."""
    effs = list(efficiencies)
    if not effs:
        raise ProtocolError("portability needs at least one device")
    if any(e <= 0.0 for e in effs):
        return 0.0
    return len(effs) / sum(1.0 / e for e in effs)


def _devices(caches: Mapping[str, TuningCache], subset) -> tuple:
    names = tuple(caches) if subset is None else tuple(subset)
    if not names:
        raise ProtocolError("the device subset is empty")
    unknown = [d for d in names if d not in caches]
    if unknown:
        raise UnknownDevice(f"no cache for device(s) {', '.join(unknown)}")
    return names


def perf_portability(caches: Mapping[str, TuningCache], subset, config) -> PortabilityReport:
    names = _devices(caches, subset)
    effs = tuple(app_efficiency(caches[d], config) for d in names)
    return PortabilityReport(names, _key(config), effs, harmonic_pp(effs))


def best_portable_config(caches: Mapping[str, TuningCache], subset=None) -> PortabilityReport:
    """argmax PP over the configurations present in every cache of the subset."""
    names = _devices(caches, subset)
    shared = set(caches[names[0]].records)
    for d in names[1:]:
        shared &= set(caches[d].records)
    if not shared:
        raise NoPortableConfiguration(f"no configuration is present in every cache of {', '.join(names)}")
    best = None
    for key in sorted(shared, key=_natural):
        report = perf_portability(caches, names, key)
        if best is None or report.pp > best.pp:
            best = report
    if best.pp <= 0.0:
        raise NoPortableConfiguration(f"every shared configuration fails on some device of {', '.join(names)}")
    return best


def write_portability_json(report: PortabilityReport, path) -> Path:
    path = Path(path)
    path.write_text(json.dumps(report.as_dict(), sort_keys=True, indent=2) + "\n", encoding="utf-8")
    return path


# ---------------------------------------------------------------------------
# Plot data


@dataclass(frozen=True)
class DistributionDataset:
    rows: tuple        # (key, metric_value, fraction_of_optimum), canonical order
    quantiles: tuple   # (percent, fraction_of_optimum)


def export_distribution(cache: TuningCache) -> DistributionDataset:
    ok = cache.ok_records()
    if not ok:
        raise _no_data(cache)
    keys = sorted(ok, key=_natural)
    perf = np.array([metric_of(ok[k]) for k in keys], dtype=np.float64)
    frac = perf / perf.max()
    rows = tuple((k, float(m), float(f)) for k, m, f in zip(keys, perf, frac))
    quant = tuple((q, float(np.percentile(frac, q))) for q in QUANTILE_PERCENTS)
    return DistributionDataset(rows, quant)


def _quote(text: str) -> str:
    return '"' + text.replace("\\", "\\\\").replace('"', '\\"') + '"'


def write_distribution_csv(dataset: DistributionDataset, path) -> Path:
    path = Path(path)
    lines = ["config_key,metric_value,fraction_of_optimum"]
    lines += [f"{_quote(k)},{m!r},{f!r}" for k, m, f in dataset.rows]
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")
    return path


def export_dot(g: FitnessFlowGraph) -> str:
    """Graphviz text; each node carries its fitness decile (0 = fastest tenth)."""
    out = ["digraph ffg {", f"  // {g.kernel_name}/{g.device_name}, scheme {g.scheme.value}, "
                            f"{g.n_nodes} nodes, {g.n_edges} edges"]
    if g.n_nodes:
        rank = np.empty(g.n_nodes, dtype=np.int64)
        rank[np.argsort(g.times, kind="stable")] = np.arange(g.n_nodes)
        bucket = np.minimum(9, (10 * rank) // g.n_nodes)
        out += [f"  {_quote(k)} [label={_quote(k)}, bucket={int(b)}];" for k, b in zip(g.keys, bucket)]
    out += [f"  {_quote(g.keys[u])} -> {_quote(g.keys[v])};" for u, v in zip(g.edge_src.tolist(),
                                                                         g.edge_dst.tolist())]
    out.append("}")
    return "\n".join(out) + "\n"
