"""Search-space sharding across the GPUs of one node (north_star N8).

One worker process per GPU (``torchrun``; RANK / LOCAL_RANK /
WORLD_SIZE from the environment), each with its own CUDA context and
:class:`CudaTarget`, pulling *chunks* of the enumeration from a dynamic
queue -- an atomic counter in the torch.distributed TCPStore -- because
per-configuration cost varies ~100x across a space (compile time and
kernel time), so static striding would leave GPUs idle.  There is no
data-path collective: configurations are independent units
(`SPEC.md:103`).  Results are gathered host-side as
``(enumeration index, key, Observation)`` and merged by index, which
reproduces the sequential brute-force trace and, through the canonical
JSON writer (sorted keys, `pkg/src/tunescape/store.py:187`), a
byte-identical cache regardless of which GPU measured what.  Ties for
the best resolve to the earliest enumeration index (ref
`strategies.py:72`).

Random search shards the same way after drawing its (timing-
independent) sequence up front (``strategies.random_sample_sequence``).

Every rank appends to its own :class:`~.store.ResultLog`; a restarted
sweep skips configurations already logged (resume after preemption).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

from .measure import BackendDescriptor, MeasurementProtocol, Observation, run_configs
from .paramspace import config_key
from .store import ResultLog, TuningCache
from .strategies import StrategyResult, result_to_cache


@dataclass
class ShardStats:
    rank: int
    configs: int
    chunks: int
    seconds: float


def dist_env() -> tuple:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ChunkQueue:
    """Dynamic chunk queue shared by all ranks (TCPStore atomic counter)."""

    def __init__(self, n_items: int, chunk: int, store=None, key: str = "tsg_next_chunk"):
        self.n, self.chunk, self.store, self.key = n_items, max(1, chunk), store, key
        self._local = 0

    def next(self):
        if self.store is None:
            i = self._local
            self._local += 1
        else:
            i = int(self.store.add(self.key, 1)) - 1
        lo = i * self.chunk
        if lo >= self.n:
            return None
        return lo, min(self.n, lo + self.chunk)


def sharded_sweep(space, configs: list, backend: BackendDescriptor, protocol: MeasurementProtocol,
                  chunk: int = 8, store=None, gather=None, log_path: str | None = None,
                  rank: int = 0, resume_from=()) -> tuple:
    """Measure ``configs`` (in order) across ranks; returns (merged trace, stats).

    ``store``: a torch.distributed Store shared by the ranks (None = one
    process); ``gather(obj) -> list`` all-gathers a picklable object
    (None = one process).  Each rank returns the full merged trace.
    ``log_path``: this rank's observation log (appended to, and resumed
    from); ``resume_from``: further logs (e.g. the other ranks' of an
    earlier run) whose observations also count as done -- the dynamic
    queue hands chunks to different ranks on a restart.
    """
    import time

    log = ResultLog(log_path) if log_path else None
    done = {}
    for extra in resume_from:
        if extra and extra != log_path:
            done.update(ResultLog(extra).load())
    if log:
        done.update(log.load())
    q = ChunkQueue(len(configs), chunk, store)
    mine: list = []
    n_chunks = 0
    t0 = time.perf_counter()
    while True:
        rng = q.next()
        if rng is None:
            break
        n_chunks += 1
        lo, hi = rng
        todo = [configs[idx] for idx in range(lo, hi) if config_key(configs[idx]) not in done]
        fresh = {}
        for c, obs in run_configs(space, backend, protocol, todo):  # cuda: pipelined
            key = config_key(c)
            fresh[key] = obs
            if log:
                log.append(key, obs)
        for idx in range(lo, hi):
            key = config_key(configs[idx])
            mine.append((idx, key, done.get(key) or fresh[key]))
    stats = ShardStats(rank, len(mine), n_chunks, time.perf_counter() - t0)
    if log:
        log.close()
    parts = gather((mine, stats)) if gather else [(mine, stats)]
    merged = sorted((item for part, _ in parts for item in part), key=lambda t: t[0])
    if len(merged) != len(configs) or any(m[0] != i for i, m in enumerate(merged)):
        raise RuntimeError("sharded sweep lost or duplicated configurations")
    return [(configs[i], obs) for i, _, obs in merged], [s for _, s in parts]


def merged_result(trace: list) -> StrategyResult:
    """StrategyResult of a merged trace (best = fastest, earliest on ties)."""
    best, best_obs = None, None
    for c, o in trace:
        if o.ok and (best_obs is None or o.time_ms < best_obs.time_ms):
            best, best_obs = c, o
    notes = () if best is not None else ("no feasible optimum: every measured configuration failed",)
    return StrategyResult(best, best_obs, tuple(trace), len(trace), notes)


def sharded_brute_force(space, backend: BackendDescriptor, protocol: MeasurementProtocol,
                        chunk: int = 8, store=None, gather=None, rank: int = 0,
                        device_name: str = "unknown", log_path: str | None = None,
                        configs: list | None = None):
    """Brute force over the whole space (or ``configs``) sharded over ranks."""
    todo = list(space.enumerate_configs()) if configs is None else list(configs)
    trace, stats = sharded_sweep(space, todo, backend, protocol, chunk, store, gather, log_path, rank)
    result = merged_result(trace)
    return result, result_to_cache(space, result, device_name), stats


def torch_dist_plumbing():
    """(store, gather, rank, world) from an initialised torch.distributed group."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return None, None, 0, 1
    from torch.distributed.distributed_c10d import _get_default_store

    store = _get_default_store()

    def gather(obj):
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, obj)
        return out

    return store, gather, dist.get_rank(), dist.get_world_size()
