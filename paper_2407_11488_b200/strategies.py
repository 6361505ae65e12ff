"""Search strategies over a space: brute force, random, greedy local, genetic.

Behavioural contract (SPEC.md ``strategies``; pinned by the reference's
tests and the golden traces in ``tests/golden``):

* fitness is the aggregated ``time_ms``, minimised; the best is the
  strictly fastest ok observation, so the earliest wins ties;
* measurements are memoised per run: revisiting a configuration costs no
  budget, and the trace records first evaluations only;
* random search draws per-parameter ``random.Random(seed).choice``,
  rejecting invalid and already-drawn points, and materialises the
  remaining valid configurations after 200 consecutive misses;
* local search is best- (or first-) improvement hill descent with random
  restarts, neighbours in parameter-then-value order, ties broken by
  canonical configuration order, the budget checked before every
  unmeasured neighbour.

Architecture (B200 build).  A strategy never measures one configuration
at a time: it hands *batches* to an :class:`Evaluator` and consumes the
observations in order.  Brute force is one batch, random search is one
batch (its draw sequence never depends on timings, so it is drawn up
front), local search batches each neighbourhood scan, and the genetic
algorithm batches each generation.  The evaluator decides how a batch
runs -- pipelined through one GPU (:class:`LocalEvaluator`, the cuda
backend's ``execute_many``), or split across the GPUs of a node
(``multigpu.ShardedEvaluator``) -- while :class:`Ledger` commits results
in the order a one-at-a-time search would have measured them, so traces,
budgets and results are identical to the sequential reference semantics
whichever evaluator runs them.  Local search's first-improvement rule
stops at the first improving neighbour; results measured past that point
are held as *speculative* and only enter the trace if the search asks
for them later.

:func:`genetic_algorithm` is new (Kernel Tuner's population search, named
by the north_star; the reference lists it as a non-goal): all its choices
come from the seeded RNG, so runs replay exactly.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .errors import ProtocolError
from .measure import BackendDescriptor, MeasurementProtocol, Observation, pipelined, run_configs
from .paramspace import Config, NeighborScheme, SearchSpaceSpec, config_key
from .store import TuningCache

MISS_LIMIT = 200  # consecutive rejected draws before sampling materialises the rest


@dataclass(frozen=True)
class SearchSegment:
    """One descent of local search: the accepted path from one start."""

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


# ---------------------------------------------------------------------------
# Evaluators: how a batch of configurations gets measured


class Evaluator:
    """Measures a list of configurations; returns their observations in order.

    ``batch_hint`` is how many configurations the evaluator can usefully
    measure at once (first-improvement local search speculates that far).
    """

    batch_hint = 1

    def measure(self, configs: list) -> list:
        raise NotImplementedError

    def device_name(self, override: str | None = None) -> str:
        return override or "unknown"


class LocalEvaluator(Evaluator):
    """One backend in this process; the cuda backend pipelines each batch."""

    def __init__(self, space: SearchSpaceSpec, backend: BackendDescriptor, protocol: MeasurementProtocol):
        self.space, self.backend, self.protocol = space, backend, protocol
        if pipelined(backend):
            self.batch_hint = max(1, int(getattr(backend.target, "pipeline_depth", 4)))

    def measure(self, configs: list) -> list:
        return [obs for _, obs in run_configs(self.space, self.backend, self.protocol, configs)]

    def device_name(self, override: str | None = None) -> str:
        return default_device_name(self.backend, override)


def default_device_name(backend: BackendDescriptor, override: str | None = None) -> str:
    """Device recorded in caches: the override, the replayed cache's device,
    the GPU's name, else ``unknown``."""
    if override:
        return override
    if backend.kind == "simulated":
        return backend.cache.device_name
    if backend.kind == "cuda":
        return backend.target.dev.info.get("name", "unknown")
    return "unknown"


# ---------------------------------------------------------------------------
# The ledger: memo, trace, best, speculative results


class Ledger:
    """Everything one strategy run has measured, in commit order."""

    def __init__(self, space: SearchSpaceSpec, evaluator: Evaluator):
        self.space, self.evaluator = space, evaluator
        self.seen: dict = {}
        self.trace: list = []
        self.best: Config | None = None
        self.best_obs: Observation | None = None
        self._speculative: dict = {}

    @property
    def evaluations(self) -> int:
        return len(self.trace)

    def lookup(self, config: Config) -> Observation | None:
        return self.seen.get(config_key(config))

    def commit(self, config: Config, obs: Observation) -> Observation:
        self.seen[config_key(config)] = obs
        self.trace.append((config, obs))
        if obs.ok and (self.best_obs is None or obs.time_ms < self.best_obs.time_ms):
            self.best, self.best_obs = config, obs
        return obs

    def unseen(self, configs) -> list:
        """``configs`` not yet committed, first occurrences, in order."""
        out, keys = [], set()
        for c in configs:
            k = config_key(c)
            if k not in self.seen and k not in keys:
                keys.add(k)
                out.append(c)
        return out

    def speculate(self, configs) -> None:
        """Measure ``configs`` now without committing them."""
        todo = [c for c in self.unseen(configs) if config_key(c) not in self._speculative]
        if todo:
            for c, obs in zip(todo, self.evaluator.measure(todo)):
                self._speculative[config_key(c)] = obs

    def take(self, config: Config) -> Observation:
        """Commit ``config`` (measured speculatively or now); memo hits are free."""
        hit = self.lookup(config)
        if hit is not None:
            return hit
        obs = self._speculative.pop(config_key(config), None)
        if obs is None:
            obs = self.evaluator.measure([config])[0]
        return self.commit(config, obs)

    def take_all(self, configs) -> None:
        """Commit a list fixed in advance: one batch, committed in order."""
        todo = self.unseen(configs)
        self.speculate(todo)
        for c in todo:
            self.take(c)

    def result(self, notes=(), segments=()) -> StrategyResult:
        notes = tuple(notes)
        if self.best is None:
            notes += ("no feasible optimum: every measured configuration failed",)
        return StrategyResult(self.best, self.best_obs, tuple(self.trace), self.evaluations, notes,
                              tuple(segments))


def _ledger(space, backend, protocol, evaluator) -> Ledger:
    if evaluator is None:
        if backend is None:
            raise ProtocolError("a strategy needs a backend or an evaluator")
        evaluator = LocalEvaluator(space, backend, protocol)
    return Ledger(space, evaluator)


def result_to_cache(space: SearchSpaceSpec, result: StrategyResult, device_name: str = "unknown",
                    metadata: dict | None = None) -> TuningCache:
    """Persistable cache of every observation a run committed."""
    return TuningCache(kernel_name=space.kernel_name, device_name=device_name,
                       param_order=space.param_names,
                       records={config_key(c): o for c, o in result.trace},
                       space_fingerprint=space.fingerprint(), provenance="native",
                       metadata=dict(metadata or {}))


# ---------------------------------------------------------------------------
# Brute force


def brute_force(space: SearchSpaceSpec, backend: BackendDescriptor | None,
                protocol: MeasurementProtocol | None, device_name: str | None = None,
                metadata: dict | None = None, configs: list | None = None,
                evaluator: Evaluator | None = None):
    """Every valid configuration once, in enumeration order (one batch).

    Returns ``(result, cache)``; the cache is complete over the space.
    ``configs`` restricts the sweep to an explicit list (a shard, a sample).
    """
    ledger = _ledger(space, backend, protocol, evaluator)
    ledger.take_all(space.enumerate_configs() if configs is None else configs)
    result = ledger.result()
    return result, result_to_cache(space, result, ledger.evaluator.device_name(device_name), metadata)


# ---------------------------------------------------------------------------
# Random search


def random_cartesian(rng: random.Random, space: SearchSpaceSpec) -> Config:
    return tuple(rng.choice(p.values) for p in space.parameters)


def random_sample_sequence(space: SearchSpaceSpec, budget: int, seed: int) -> tuple:
    """``(configs, notes)``: the draws :func:`random_search` commits, in order.

    Draws depend only on the seed and on which configurations were drawn
    before -- never on timings -- so the sequence is the whole plan.
    """
    if budget < 1:
        raise ProtocolError("random search needs a budget of at least 1")
    rng = random.Random(seed)
    drawn: dict = {}
    notes: list = []
    rest: list | None = None
    misses = 0
    while len(drawn) < budget:
        if rest is None:
            cand = random_cartesian(rng, space)
            if config_key(cand) in drawn or not space.satisfies(cand):
                misses += 1
                if misses >= MISS_LIMIT:
                    rest = [c for c in space.enumerate_configs() if config_key(c) not in drawn]
                continue
            misses = 0
        elif rest:
            cand = rest.pop(rng.randrange(len(rest)))
        else:
            notes.append(f"budget {budget} clamped to space size {len(drawn)}")
            break
        drawn[config_key(cand)] = cand
    return list(drawn.values()), notes


def random_search(space: SearchSpaceSpec, backend: BackendDescriptor | None,
                  protocol: MeasurementProtocol | None, budget: int, seed: int,
                  evaluator: Evaluator | None = None) -> StrategyResult:
    """Uniform sampling without replacement (seeded, replayable; one batch)."""
    plan, notes = random_sample_sequence(space, budget, seed)
    ledger = _ledger(space, backend, protocol, evaluator)
    ledger.take_all(plan)
    return ledger.result(notes=notes)


# ---------------------------------------------------------------------------
# Greedy local search


class _Starts:
    """Random valid starting points (rejection sampling, then a pool)."""

    def __init__(self, space: SearchSpaceSpec, rng: random.Random):
        self.space, self.rng, self.pool = space, rng, None

    def draw(self) -> Config | None:
        misses = 0
        while self.pool is None:
            cand = random_cartesian(self.rng, self.space)
            if self.space.satisfies(cand):
                return cand
            misses += 1
            if misses >= MISS_LIMIT:
                self.pool = list(self.space.enumerate_configs())
        return self.pool[self.rng.randrange(len(self.pool))] if self.pool else None


def _scan(ledger: Ledger, here_ms: float, neighbours: list, budget: int, first_improvement: bool,
          order_of) -> tuple:
    """One neighbourhood scan: ``(move, out_of_budget)``.

    Commits neighbours in neighbour order exactly as a one-at-a-time scan
    would -- an unmeasured neighbour met with the budget spent ends the
    scan -- but measures them in batches.  Best-improvement measures every
    affordable neighbour as one batch; first-improvement speculates
    ``batch_hint`` neighbours ahead and stops committing at the first
    improvement.
    """
    fresh = ledger.unseen(neighbours)
    affordable = fresh[:max(0, budget - ledger.evaluations)]
    window = len(affordable) if not first_improvement else max(1, ledger.evaluator.batch_hint)
    pos = {config_key(c): i for i, c in enumerate(affordable)}
    move, move_ms = None, None
    for cand in neighbours:
        key = config_key(cand)
        if ledger.lookup(cand) is None:
            if ledger.evaluations >= budget:
                return None, True
            i = pos[key]
            if i % window == 0:
                ledger.speculate(affordable[i:i + window])
        obs = ledger.take(cand)
        if not obs.ok or obs.time_ms >= here_ms:
            continue
        if first_improvement:
            return cand, False
        if move is None or obs.time_ms < move_ms or (obs.time_ms == move_ms and order_of(cand) < order_of(move)):
            move, move_ms = cand, obs.time_ms
    return move, False


def greedy_local_search(space: SearchSpaceSpec, backend: BackendDescriptor | None,
                        protocol: MeasurementProtocol | None, budget: int, seed: int,
                        scheme: NeighborScheme | str | None = None,
                        first_improvement: bool = False,
                        start: Config | None = None,
                        evaluator: Evaluator | None = None) -> StrategyResult:
    """Hill descent with random restarts; each neighbourhood is one batch."""
    if budget < 1:
        raise ProtocolError("local search needs a budget of at least 1")
    scheme = NeighborScheme(scheme) if scheme else space.neighbor_scheme
    ledger = _ledger(space, backend, protocol, evaluator)
    starts = _Starts(space, random.Random(seed))
    segments, notes = [], []
    size = None
    pending_start = start
    while ledger.evaluations < budget:
        origin, pending_start = (pending_start or starts.draw()), None
        if origin is None:
            notes.append("space has no valid configurations")
            break
        before = ledger.evaluations
        path, here = [origin], origin
        here_obs = ledger.take(origin)
        at_minimum = out_of_budget = False
        while here_obs.ok:
            move, out_of_budget = _scan(ledger, here_obs.time_ms, space.neighbors(here, scheme), budget,
                                        first_improvement, space.flat_index)
            if out_of_budget:
                break
            if move is None:
                at_minimum = True
                break
            here, here_obs = move, ledger.lookup(move)
            path.append(here)
        segments.append(SearchSegment(tuple(path), at_minimum))
        if out_of_budget or ledger.evaluations >= budget:
            break
        if ledger.evaluations == before:  # a restart that measured nothing new
            size = space.space_size() if size is None else size
            if len(ledger.seen) >= size:
                notes.append("entire space evaluated before budget ran out")
                break
    return ledger.result(notes=notes, segments=segments)


# ---------------------------------------------------------------------------
# Genetic algorithm (new; Kernel Tuner's strategy="genetic_algorithm")

_CROSSOVERS = ("uniform", "single_point", "two_point")


def genetic_algorithm(space: SearchSpaceSpec, backend: BackendDescriptor | None,
                      protocol: MeasurementProtocol | None, budget: int, seed: int,
                      popsize: int = 20, maxiter: int = 100, mutation_chance: int = 10,
                      crossover: str = "uniform", evaluator: Evaluator | None = None) -> StrategyResult:
    """Population search over valid configurations; one batch per generation.

    * the first generation is ``popsize`` distinct valid random points;
    * rank selection (weight ``popsize - rank``; failures rank last), the
      top tenth survives unchanged (elitism), ``crossover`` in
      {uniform, single_point, two_point}, per-gene mutation with
      probability ``1/mutation_chance``; an invalid child is re-mutated up
      to 100 times, then replaced by a random valid point;
    * stops at ``budget`` distinct evaluations, ``maxiter`` generations or
      an exhausted space.
    """
    if budget < 1:
        raise ProtocolError("genetic algorithm needs a budget of at least 1")
    if crossover not in _CROSSOVERS:
        raise ProtocolError(f"unknown crossover {crossover!r}; one of {', '.join(_CROSSOVERS)}")
    rng = random.Random(seed)
    ledger = _ledger(space, backend, protocol, evaluator)
    size = space.space_size()
    width = len(space.parameters)

    def random_valid() -> Config | None:
        for _ in range(10 * MISS_LIMIT):
            cand = random_cartesian(rng, space)
            if space.satisfies(cand):
                return cand
        pool = list(space.enumerate_configs())
        return pool[rng.randrange(len(pool))] if pool else None

    def mutate(genes: Config) -> Config:
        return tuple(rng.choice(p.values) if rng.randrange(mutation_chance) == 0 else g
                     for g, p in zip(genes, space.parameters))

    def recombine(a: Config, b: Config) -> Config:
        if crossover == "uniform":
            return tuple(x if rng.random() < 0.5 else y for x, y in zip(a, b))
        if crossover == "single_point":
            cut = rng.randrange(1, width) if width > 1 else 0
            return a[:cut] + b[cut:]
        lo, hi = sorted(rng.sample(range(width + 1), 2))
        return a[:lo] + b[lo:hi] + a[hi:]

    def repaired(child: Config) -> Config | None:
        for _ in range(100):
            if space.satisfies(child):
                return child
            child = mutate(child)
        return child if space.satisfies(child) else random_valid()

    def fitness(c: Config) -> float:
        obs = ledger.lookup(c)
        return obs.time_ms if obs is not None and obs.ok else float("inf")

    population: dict = {}
    while len(population) < min(popsize, size):
        cand = random_valid()
        if cand is None:
            break
        population.setdefault(config_key(cand), cand)
    population = list(population.values())

    notes = []
    generation = 0
    while ledger.evaluations < budget and generation < maxiter:
        ledger.take_all(ledger.unseen(population)[:budget - ledger.evaluations])
        if len(ledger.seen) >= size:
            notes.append("entire space evaluated before budget ran out")
            break
        ranked = sorted(population, key=lambda c: (fitness(c), config_key(c)))
        weights = list(range(len(ranked), 0, -1))
        elite = ranked[:max(1, len(ranked) // 10)]
        children = {config_key(c): c for c in elite}
        attempts = 0
        while len(children) < popsize and attempts < 50 * popsize:
            attempts += 1
            mum, dad = rng.choices(ranked, weights=weights, k=2)
            child = repaired(mutate(recombine(mum, dad)))
            key = config_key(child)
            if key in children:
                continue
            if ledger.lookup(child) is not None and attempts < 25 * popsize:
                continue  # prefer unexplored children until the population converges
            children[key] = child
        population = list(children.values())
        generation += 1
    if generation >= maxiter:
        notes.append(f"stopped after {maxiter} generations")
    return ledger.result(notes=notes)


STRATEGIES = {
    "brute_force": brute_force,
    "random_sample": random_search,
    "random": random_search,
    "greedy_ls": greedy_local_search,
    "local": greedy_local_search,
    "genetic_algorithm": genetic_algorithm,
    "genetic": genetic_algorithm,
}
