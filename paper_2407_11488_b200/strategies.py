"""Search strategies: brute force, random, greedy local search, genetic.

Semantics follow the reference (`pkg/src/tunescape/strategies.py`):
fitness is the aggregated ``time_ms`` (minimised); a memoising runner
(:45-87) makes revisits free; the best is the strictly fastest ok
observation, so the earliest wins ties (:72); ``random_search`` draws
per-parameter ``random.Random(seed).choice`` with rejection of invalid
or seen points and materialises the remainder after 200 misses
(:148-192); ``greedy_local_search`` scans neighbours in parameter/value
order with canonical tie-breaks and random restarts (:195-297).  With
the same seed the traces are identical to the reference's.

B200 additions:
* with a ``cuda`` backend the runner pipelines NVRTC compilation ahead
  of the GPU (``target.prefetch``), because compile, not the kernel,
  bounds configurations/second;
* :func:`genetic_algorithm` (absent from the reference; Kernel Tuner's
  population-based search, north_star) -- selection, crossover and
  mutation draw only from the seeded RNG, so runs are replayable.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .errors import ProtocolError
from .measure import BackendDescriptor, MeasurementProtocol, Observation, pipelined, run_config, run_configs
from .paramspace import Config, NeighborScheme, SearchSpaceSpec, config_key
from .store import TuningCache

MISS_LIMIT = 200


@dataclass(frozen=True)
class SearchSegment:
    path: tuple
    reached_minimum: bool


@dataclass(frozen=True)
class StrategyResult:
    best: Config | None
    best_observation: Observation | None
    trace: tuple
    evaluations_used: int
    notes: tuple = ()
    segments: tuple = ()


class Runner:
    """Memoising measurement driver shared by every strategy."""

    def __init__(self, space: SearchSpaceSpec, backend: BackendDescriptor,
                 protocol: MeasurementProtocol):
        self.space, self.backend, self.protocol = space, backend, protocol
        self.seen: dict = {}
        self.trace: list = []
        self.best: Config | None = None
        self.best_obs: Observation | None = None

    @property
    def evaluations(self) -> int:
        return len(self.trace)

    def lookup(self, config: Config):
        return self.seen.get(config_key(config))

    def prefetch(self, configs) -> None:
        if self.backend.kind == "cuda":
            self.backend.target.prefetch(c for c in configs if config_key(c) not in self.seen)

    def record(self, config: Config, obs: Observation) -> Observation:
        key = config_key(config)
        self.seen[key] = obs
        self.trace.append((config, obs))
        if obs.ok and (self.best_obs is None or obs.time_ms < self.best_obs.time_ms):
            self.best, self.best_obs = config, obs
        return obs

    def evaluate(self, config: Config) -> Observation:
        hit = self.seen.get(config_key(config))
        if hit is not None:
            return hit
        return self.record(config, run_config(self.space, self.backend, self.protocol, config))

    def evaluate_many(self, configs) -> None:
        """Evaluate a list fixed in advance, in order (memoised; the cuda
        backend pipelines it -- same trace as evaluating one by one)."""
        todo, keys = [], set()
        for c in configs:
            k = config_key(c)
            if k not in self.seen and k not in keys:
                keys.add(k)
                todo.append(c)
        for c, obs in run_configs(self.space, self.backend, self.protocol, todo):
            self.record(c, obs)

    def result(self, notes=(), segments=()) -> StrategyResult:
        notes = tuple(notes)
        if self.best is None:
            notes += ("no feasible optimum: every measured configuration failed",)
        return StrategyResult(self.best, self.best_obs, tuple(self.trace), self.evaluations,
                              notes, tuple(segments))


# kept for callers written against the reference's private name
_Runner = Runner


def result_to_cache(space: SearchSpaceSpec, result: StrategyResult, device_name: str = "unknown",
                    metadata: dict | None = None) -> TuningCache:
    return TuningCache(kernel_name=space.kernel_name, device_name=device_name,
                       param_order=space.param_names,
                       records={config_key(c): o for c, o in result.trace},
                       space_fingerprint=space.fingerprint(), provenance="native",
                       metadata=dict(metadata or {}))


def default_device_name(backend: BackendDescriptor, override: str | None = None) -> str:
    if override:
        return override
    if backend.kind == "simulated":
        return backend.cache.device_name
    if backend.kind == "cuda":
        return backend.target.dev.info.get("name", "unknown")
    return "unknown"


def _window(runner: Runner, configs: list, start: int) -> None:
    if runner.backend.kind == "cuda":
        depth = runner.backend.target.prefetch_depth
        runner.prefetch(configs[start:start + depth])


def brute_force(space: SearchSpaceSpec, backend: BackendDescriptor,
                protocol: MeasurementProtocol, device_name: str | None = None,
                metadata: dict | None = None, configs: list | None = None):
    """Measure every valid configuration once, in enumeration order.

    ``configs`` (new) restricts the sweep to an explicit sub-list, in the
    given order -- the unit a multi-GPU shard runs.
    """
    runner = Runner(space, backend, protocol)
    todo = list(space.enumerate_configs()) if configs is None else list(configs)
    if pipelined(backend):
        runner.evaluate_many(todo)  # pipelined, same order
    else:
        for i, config in enumerate(todo):
            if i % 8 == 0:
                _window(runner, todo, i)
            runner.evaluate(config)
    result = runner.result()
    return result, result_to_cache(space, result, default_device_name(backend, device_name),
                                   metadata)


def random_cartesian(rng: random.Random, space: SearchSpaceSpec) -> Config:
    return tuple(rng.choice(p.values) for p in space.parameters)


def random_sample_sequence(space: SearchSpaceSpec, budget: int, seed: int) -> tuple:
    """The configurations random_search would evaluate, and its notes.

    The sequence never depends on measured times (ref :170-191), so it
    can be drawn up front and sharded across GPUs while keeping the
    trace identical to the sequential run.
    """
    if budget < 1:
        raise ProtocolError("random search needs a budget of at least 1")
    rng = random.Random(seed)
    seen: set = set()
    order: list = []
    notes: list = []
    remaining = None
    misses = 0
    while len(order) < budget:
        if remaining is None:
            config = random_cartesian(rng, space)
            key = config_key(config)
            if not space.satisfies(config) or key in seen:
                misses += 1
                if misses >= MISS_LIMIT:
                    remaining = [c for c in space.enumerate_configs() if config_key(c) not in seen]
                continue
            misses = 0
        else:
            if not remaining:
                notes.append(f"budget {budget} clamped to space size {len(order)}")
                break
            config = remaining.pop(rng.randrange(len(remaining)))
            key = config_key(config)
        seen.add(key)
        order.append(config)
    return order, notes


def random_search(space: SearchSpaceSpec, backend: BackendDescriptor,
                  protocol: MeasurementProtocol, budget: int, seed: int) -> StrategyResult:
    """Uniform sampling without replacement (seeded, replayable)."""
    order, notes = random_sample_sequence(space, budget, seed)
    runner = Runner(space, backend, protocol)
    if pipelined(backend):
        runner.evaluate_many(order)  # the order is timing-independent: pipelined
    else:
        for i, config in enumerate(order):
            if i % 8 == 0:
                _window(runner, order, i)
            runner.evaluate(config)
    return runner.result(notes=notes)


def greedy_local_search(space: SearchSpaceSpec, backend: BackendDescriptor,
                        protocol: MeasurementProtocol, budget: int, seed: int,
                        scheme: NeighborScheme | str | None = None,
                        first_improvement: bool = False,
                        start: Config | None = None) -> StrategyResult:
    """Hill descent with random restarts (ref strategies.py:195-297)."""
    if budget < 1:
        raise ProtocolError("local search needs a budget of at least 1")
    scheme = NeighborScheme(scheme) if scheme else space.neighbor_scheme
    rng = random.Random(seed)
    runner = Runner(space, backend, protocol)
    segments: list = []
    notes: list = []
    pool = None
    size = None
    pos = [{v: i for i, v in enumerate(p.values)} for p in space.parameters]

    def rank(c):
        return tuple(m[v] for m, v in zip(pos, c))

    def fresh_start():
        nonlocal pool
        misses = 0
        while pool is None:
            cand = random_cartesian(rng, space)
            if space.satisfies(cand):
                return cand
            misses += 1
            if misses >= MISS_LIMIT:
                pool = list(space.enumerate_configs())
        return pool[rng.randrange(len(pool))] if pool else None

    first = True
    while runner.evaluations < budget:
        origin = start if (first and start is not None) else fresh_start()
        first = False
        if origin is None:
            notes.append("space has no valid configurations")
            break
        before = runner.evaluations
        path = [origin]
        cur_obs = runner.evaluate(origin)
        cur = origin
        at_min = False
        exhausted = False
        while cur_obs.ok:
            nbrs = space.neighbors(cur, scheme)
            runner.prefetch(nbrs)
            move, move_t = None, None
            for cand in nbrs:
                if runner.lookup(cand) is None and runner.evaluations >= budget:
                    exhausted = True
                    break
                o = runner.evaluate(cand)
                if not o.ok or o.time_ms >= cur_obs.time_ms:
                    continue
                if first_improvement:
                    move, move_t = cand, o.time_ms
                    break
                if move is None or o.time_ms < move_t or (o.time_ms == move_t and rank(cand) < rank(move)):
                    move, move_t = cand, o.time_ms
            if exhausted:
                break
            if move is None:
                at_min = True
                break
            cur = move
            cur_obs = runner.seen[config_key(cur)]
            path.append(cur)
        segments.append(SearchSegment(tuple(path), at_min))
        if exhausted or runner.evaluations >= budget:
            break
        if runner.evaluations == before:
            if size is None:
                size = space.space_size()
            if len(runner.seen) >= size:
                notes.append("entire space evaluated before budget ran out")
                break
    return runner.result(notes=notes, segments=segments)


# -----------------------------------------------------------------------------
# Genetic algorithm (new; Kernel Tuner's strategy="genetic_algorithm")


def genetic_algorithm(space: SearchSpaceSpec, backend: BackendDescriptor,
                      protocol: MeasurementProtocol, budget: int, seed: int,
                      popsize: int = 20, maxiter: int = 100, mutation_chance: int = 10,
                      crossover: str = "uniform", evaluate_population=None) -> StrategyResult:
    """Population search over valid configurations.

    * initial population: ``popsize`` distinct valid points (rejection
      sampling like :func:`random_search`);
    * each generation is evaluated as a batch (``evaluate_population``
      may fan it out over several GPUs; default: sequential, memoised);
    * rank selection (weight ~ popsize - rank), ``crossover`` in
      {uniform, single_point, two_point}, per-gene mutation with
      probability 1/mutation_chance; invalid children are repaired by
      re-mutating up to 100 times, else replaced by a random point;
    * failed configurations rank last; stops at ``budget`` distinct
      evaluations, ``maxiter`` generations, or space exhaustion.
    """
    if budget < 1:
        raise ProtocolError("genetic algorithm needs a budget of at least 1")
    if crossover not in ("uniform", "single_point", "two_point"):
        raise ProtocolError(f"unknown crossover {crossover!r}")
    rng = random.Random(seed)
    runner = Runner(space, backend, protocol)
    notes: list = []
    n_params = len(space.parameters)
    size = space.space_size()

    def random_valid():
        for _ in range(10 * MISS_LIMIT):
            c = random_cartesian(rng, space)
            if space.satisfies(c):
                return c
        pool = list(space.enumerate_configs())
        return pool[rng.randrange(len(pool))] if pool else None

    def mutate(c):
        genes = list(c)
        for i, p in enumerate(space.parameters):
            if rng.randrange(mutation_chance) == 0:
                genes[i] = rng.choice(p.values)
        return tuple(genes)

    def cross(a, b):
        if crossover == "uniform":
            return tuple(x if rng.random() < 0.5 else y for x, y in zip(a, b))
        if crossover == "single_point":
            k = rng.randrange(1, n_params) if n_params > 1 else 0
            return a[:k] + b[k:]
        i, j = sorted(rng.sample(range(n_params + 1), 2))
        return a[:i] + b[i:j] + a[j:]

    def fitness(c):
        o = runner.lookup(c)
        return o.time_ms if (o is not None and o.ok) else float("inf")

    population = []
    keys = set()
    while len(population) < min(popsize, size):
        c = random_valid()
        if c is None:
            break
        if config_key(c) not in keys:
            keys.add(config_key(c))
            population.append(c)

    gen = 0
    while runner.evaluations < budget and gen < maxiter:
        todo = [c for c in population if runner.lookup(c) is None]
        todo = todo[: budget - runner.evaluations]
        if evaluate_population is not None and todo:
            for c, o in zip(todo, evaluate_population(todo)):
                if runner.lookup(c) is None:
                    runner.record(c, o)
        else:
            runner.prefetch(todo)
            for c in todo:
                runner.evaluate(c)
        if len(runner.seen) >= size:
            notes.append("entire space evaluated before budget ran out")
            break
        ranked = sorted(population, key=lambda c: (fitness(c), config_key(c)))
        weights = [len(ranked) - i for i in range(len(ranked))]
        children = []
        child_keys = set()
        elite = ranked[: max(1, len(ranked) // 10)]
        for e in elite:
            children.append(e)
            child_keys.add(config_key(e))
        attempts = 0
        while len(children) < popsize and attempts < 50 * popsize:
            attempts += 1
            pa, pb = rng.choices(ranked, weights=weights, k=2)
            child = mutate(cross(pa, pb))
            tries = 0
            while not space.satisfies(child) and tries < 100:
                child = mutate(child)
                tries += 1
            if not space.satisfies(child):
                child = random_valid()
            k = config_key(child)
            if k in child_keys:
                continue
            # prefer unexplored children once the population has converged
            if runner.lookup(child) is not None and attempts < 25 * popsize:
                continue
            child_keys.add(k)
            children.append(child)
        population = children
        gen += 1
    if gen >= maxiter:
        notes.append(f"stopped after {maxiter} generations")
    return runner.result(notes=notes)


STRATEGIES = {
    "brute_force": brute_force,
    "random_sample": random_search,
    "random": random_search,
    "greedy_ls": greedy_local_search,
    "local": greedy_local_search,
    "genetic_algorithm": genetic_algorithm,
    "genetic": genetic_algorithm,
}
