"""Strategy parity with the reference (golden traces) + the new GA.

For each golden random space the reference ran brute force, random
search and greedy local search over a simulated (replay) backend; the
traces, best configurations, notes and segments must be identical here
(`pkg/src/tunescape/strategies.py:117-297`), and brute force must
produce the byte-identical canonical cache (`store.py:174-187`).
"""

import pytest

from paper_2407_11488_b200.measure import MeasurementProtocol, Observation, Status, simulated_backend
from paper_2407_11488_b200.paramspace import bundled_space, config_key, parse_space_spec
from paper_2407_11488_b200.store import TuningCache, dumps_cache
from paper_2407_11488_b200.strategies import (
    brute_force,
    genetic_algorithm,
    greedy_local_search,
    random_sample_sequence,
    random_search,
)


def golden_backend(rec):
    s = parse_space_spec(rec["text"])
    records = {}
    for key, (status, t) in rec["records"].items():
        c = s.config_from_key(key)
        if status == "ok":
            records[key] = Observation(Status.OK, (t,), t, s.metric_value(t, c))
        else:
            records[key] = Observation(Status(status))
    cache = TuningCache(kernel_name=s.kernel_name, device_name="devA", param_order=s.param_names,
                        records=records, space_fingerprint=s.fingerprint())
    return s, simulated_backend(cache)


def test_golden_traces(golden):
    proto = MeasurementProtocol()
    n = 0
    for rec in golden["strategies"]:
        s, be = golden_backend(rec)
        bf, cache = brute_force(s, be, proto)
        assert (config_key(bf.best) if bf.best else None) == rec["brute_best"]
        assert dumps_cache(cache) == rec["cache_text"]
        for run in rec["runs"]:
            if run["kind"] == "random":
                r = random_search(s, be, proto, budget=run["budget"], seed=run["seed"])
            elif run["kind"] == "greedy":
                r = greedy_local_search(s, be, proto, budget=run["budget"], seed=run["seed"])
                assert [[list(map(config_key, sg.path)), sg.reached_minimum] for sg in r.segments] \
                    == run["segments"]
            else:
                r = greedy_local_search(s, be, proto, budget=run["budget"], seed=run["seed"],
                                        first_improvement=True, scheme="adjacent")
            assert [config_key(c) for c, _ in r.trace] == run["trace"], run["kind"]
            assert list(r.notes) == run["notes"]
            assert (config_key(r.best) if r.best else None) == run["best"]
            n += 1
    assert n > 100


def test_random_sequence_independent_of_times(golden):
    rec = golden["strategies"][0]
    s, be = golden_backend(rec)
    order, _ = random_sample_sequence(s, 5, 7)
    r = random_search(s, be, MeasurementProtocol(), budget=5, seed=7)
    assert [c for c, _ in r.trace] == order


def _synthetic_backend(space, seed=0):
    import random

    rng = random.Random(seed)
    recs = {}
    for c in space.enumerate_configs():
        t = round(rng.uniform(0.1, 100), 6)
        recs[config_key(c)] = Observation(Status.OK, (t,), t)
    cache = TuningCache(kernel_name=space.kernel_name, device_name="d", param_order=space.param_names,
                        records=recs, space_fingerprint=space.fingerprint())
    return simulated_backend(cache), recs


def test_genetic_is_deterministic_and_valid():
    space = bundled_space("convolution")
    be, recs = _synthetic_backend(space)
    a = genetic_algorithm(space, be, MeasurementProtocol(), budget=200, seed=3)
    b = genetic_algorithm(space, be, MeasurementProtocol(), budget=200, seed=3)
    assert [c for c, _ in a.trace] == [c for c, _ in b.trace]
    assert len(a.trace) == 200 == a.evaluations_used
    assert all(space.is_valid(c) for c, _ in a.trace)
    assert len({config_key(c) for c, _ in a.trace}) == 200
    best_t = min(o.time_ms for _, o in a.trace)
    assert a.best_observation.time_ms == best_t


def test_genetic_beats_random_on_average():
    space = bundled_space("dedispersion")
    # smooth landscape: time grows with distance from a target configuration
    target = list(space.enumerate_configs())[5000]
    recs = {}
    for c in space.enumerate_configs():
        d = sum(abs(space.parameters[i].values.index(v) - space.parameters[i].values.index(target[i]))
                for i, v in enumerate(c))
        recs[config_key(c)] = Observation(Status.OK, (1.0 + d,), 1.0 + d)
    cache = TuningCache("dedispersion", "d", space.param_names, recs, space.fingerprint())
    be = simulated_backend(cache)
    ga = [genetic_algorithm(space, be, MeasurementProtocol(), budget=150, seed=s).best_observation.time_ms
          for s in range(6)]
    rs = [random_search(space, be, MeasurementProtocol(), budget=150, seed=s).best_observation.time_ms
          for s in range(6)]
    assert sum(ga) < sum(rs)


def test_genetic_exhausts_small_space():
    from paper_2407_11488_b200.paramspace import space_from_tune_params

    space = space_from_tune_params("tiny", {"a": [1, 2, 3], "b": [1, 2]})
    be, _ = _synthetic_backend(space)
    r = genetic_algorithm(space, be, MeasurementProtocol(), budget=100, seed=0, popsize=4)
    assert len(r.trace) == 6
    assert "entire space evaluated before budget ran out" in r.notes


def test_budget_validation():
    from paper_2407_11488_b200.errors import ProtocolError

    space = bundled_space("convolution")
    be, _ = _synthetic_backend(space)
    with pytest.raises(ProtocolError):
        random_search(space, be, MeasurementProtocol(), budget=0, seed=0)
    with pytest.raises(ProtocolError):
        genetic_algorithm(space, be, MeasurementProtocol(), budget=0, seed=0)
