"""Strategies across the GPUs of one node (north_star: "the search space is
partitioned across the 8 GPUs of one B200 box").

One worker process per GPU (``torchrun``; RANK / LOCAL_RANK / WORLD_SIZE
from the environment), each with its own CUDA context and
:class:`~.cuda_backend.CudaTarget`.  Every rank runs the *same* strategy
code with the same seed (SPMD): whenever the strategy hands a batch to its
evaluator, :class:`ShardedEvaluator` splits the batch over the ranks and
all-gathers the observations, so every rank sees identical results, takes
identical decisions and commits identical traces.  That gives all four
strategies a multi-GPU form with no master process:

* brute force -- the whole space is one batch;
* random search -- the (timing-independent) draw sequence is one batch;
* local search -- each neighbourhood scan is a batch (the budget cut and
  the canonical tie-break are applied by the ledger, in neighbour order);
* genetic -- each generation is a batch.

Within a batch, ranks pull *chunks* from a dynamic queue -- an atomic
counter in the torch.distributed TCPStore, one counter per batch --
because per-configuration cost varies ~100x across a space (compile and
kernel time); static striding would leave GPUs idle.  There is no
data-path collective: configurations are independent units
(SURVEY §8e).  Results travel host-side as (batch index, Observation)
and are merged by index, which reproduces the sequential trace and,
through the canonical JSON writer, a byte-identical cache.

Every rank may append what it measured to its own :class:`~.store.ResultLog`
(``<log>.rank<N>``); a restarted run counts observations in any earlier
log as done (the dynamic queue hands chunks to different ranks on a
restart).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

from .measure import BackendDescriptor, MeasurementProtocol, run_configs
from .paramspace import config_key
from .store import ResultLog
from .strategies import Evaluator, Ledger, StrategyResult, default_device_name, result_to_cache


@dataclass
class ShardStats:
    rank: int
    configs: int
    chunks: int
    seconds: float


def dist_env() -> tuple:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


@dataclass
class Comm:
    """Host-side plumbing between the ranks of one job."""

    store: object = None   # torch.distributed Store (None: one process)
    gather: object = None  # all-gather of a picklable object (None: one process)
    rank: int = 0
    world: int = 1


def torch_dist_plumbing():
    """(store, gather, rank, world) from an initialised torch.distributed group."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return None, None, 0, 1
    from torch.distributed.distributed_c10d import _get_default_store

    def gather(obj):
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, obj)
        return out

    return _get_default_store(), gather, dist.get_rank(), dist.get_world_size()


def current_comm() -> Comm:
    return Comm(*torch_dist_plumbing())


class ChunkQueue:
    """Dynamic chunk queue over ``n_items`` shared by all ranks."""

    def __init__(self, n_items: int, chunk: int, store=None, key: str = "tsg_next_chunk"):
        self.n, self.chunk, self.store, self.key = n_items, max(1, chunk), store, key
        self._local = 0

    def next(self):
        if self.store is None:
            ticket, self._local = self._local, self._local + 1
        else:
            ticket = int(self.store.add(self.key, 1)) - 1
        lo = ticket * self.chunk
        return None if lo >= self.n else (lo, min(self.n, lo + self.chunk))


class ShardedEvaluator(Evaluator):
    """Splits every batch over the ranks; every rank gets all observations.

    ``log_path``: this rank's observation log (appended to; its entries
    count as done); ``resume_from``: more logs whose entries count as done.
    """

    _instances = 0  # same count on every rank (SPMD): names this evaluator's queues

    def __init__(self, space, backend: BackendDescriptor, protocol: MeasurementProtocol,
                 comm: Comm | None = None, chunk: int = 8, log_path: str | None = None,
                 resume_from=(), space_check: bool = True):
        ShardedEvaluator._instances += 1
        self.tag = f"tsg_ev{ShardedEvaluator._instances}"
        self.space, self.backend, self.protocol = space, backend, protocol
        self.comm = comm or Comm()
        self.chunk = max(1, chunk)
        self.batches = 0
        self.stats = ShardStats(self.comm.rank, 0, 0, 0.0)
        self.all_stats: list = []
        hdr = dict(space=space, protocol=protocol) if space_check else {}
        self.log = ResultLog(log_path, **hdr) if log_path else None
        self.done: dict = {}
        for extra in resume_from:
            if extra and extra != log_path:
                self.done.update(ResultLog(extra, **hdr).load())
        if self.log is not None:
            self.done.update(self.log.load())
        depth = getattr(getattr(backend, "target", None), "pipeline_depth", 1)
        self.batch_hint = max(1, self.comm.world * (depth if backend.kind == "cuda" else 1))

    def device_name(self, override: str | None = None) -> str:
        return default_device_name(self.backend, override)

    def measure(self, configs: list) -> list:
        configs = list(configs)
        self.batches += 1
        queue = ChunkQueue(len(configs), self.chunk, self.comm.store, key=f"{self.tag}_batch{self.batches}")
        mine: list = []
        t0 = time.perf_counter()
        while True:
            span = queue.next()
            if span is None:
                break
            self.stats.chunks += 1
            lo, hi = span
            todo = [c for c in configs[lo:hi] if config_key(c) not in self.done]
            fresh = {}
            for c, obs in run_configs(self.space, self.backend, self.protocol, todo):  # cuda: pipelined
                fresh[config_key(c)] = obs
                if self.log is not None:
                    self.log.append(config_key(c), obs)
            for idx in range(lo, hi):
                key = config_key(configs[idx])
                mine.append((idx, self.done.get(key) or fresh[key]))
        self.stats.configs += len(mine)
        self.stats.seconds += time.perf_counter() - t0
        parts = self.comm.gather((mine, self.stats)) if self.comm.gather else [(mine, self.stats)]
        self.all_stats = [s for _, s in parts]
        merged = sorted((item for part, _ in parts for item in part), key=lambda t: t[0])
        if [i for i, _ in merged] != list(range(len(configs))):
            raise RuntimeError("a sharded batch lost or duplicated configurations")
        return [obs for _, obs in merged]

    def close(self) -> None:
        if self.log is not None:
            self.log.close()


def sharded_sweep(space, configs: list, backend: BackendDescriptor, protocol: MeasurementProtocol,
                  chunk: int = 8, store=None, gather=None, log_path: str | None = None,
                  rank: int = 0, resume_from=()) -> tuple:
    """Measure ``configs`` (one batch) across ranks; ``(trace, per-rank stats)``.

    Every rank returns the full merged trace in ``configs`` order.
    """
    world = 1 if gather is None else len(gather(None))
    ev = ShardedEvaluator(space, backend, protocol, Comm(store, gather, rank, world), chunk, log_path,
                          resume_from)
    try:
        observations = ev.measure(configs)
    finally:
        ev.close()
    return list(zip(configs, observations)), ev.all_stats


def merged_result(trace: list) -> StrategyResult:
    """StrategyResult of a merged trace (best = fastest, earliest on ties)."""
    ledger = Ledger(None, Evaluator())
    for config, obs in trace:
        ledger.commit(config, obs)
    return ledger.result()


def sharded_brute_force(space, backend: BackendDescriptor, protocol: MeasurementProtocol,
                        chunk: int = 8, store=None, gather=None, rank: int = 0,
                        device_name: str = "unknown", log_path: str | None = None,
                        configs: list | None = None):
    """Brute force over the whole space (or ``configs``) sharded over ranks."""
    todo = list(space.enumerate_configs()) if configs is None else list(configs)
    trace, stats = sharded_sweep(space, todo, backend, protocol, chunk, store, gather, log_path, rank)
    result = merged_result(trace)
    return result, result_to_cache(space, result, device_name), stats
