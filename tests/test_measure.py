"""Measurement boundary (ref `pkg/tests/test_measure.py` strategy).

The command backend keeps the reference's stdout contract; the new
``cuda`` kind is an in-process executor and ``gpu`` stays rejected.
"""

import sys
import textwrap

import pytest

from paper_2407_11488_b200.errors import EvaluationError, MissingEntry, ProtocolError
from paper_2407_11488_b200.measure import (
    BackendDescriptor,
    MeasurementProtocol,
    Observation,
    Status,
    command_backend,
    compute_metric,
    measure,
    run_config,
    simulated_backend,
)
from paper_2407_11488_b200.paramspace import bundled_space, space_from_tune_params
from paper_2407_11488_b200.store import TuningCache


def test_protocol_defaults_match_reference():
    p = MeasurementProtocol()
    assert (p.warmup_runs, p.benchmark_runs, p.aggregate.value, p.timeout_ms) == (1, 7, "mean", 60000.0)
    with pytest.raises(ProtocolError):
        MeasurementProtocol(benchmark_runs=0)
    with pytest.raises(ProtocolError):
        MeasurementProtocol(warmup_runs=-1)


def test_observation_invariants():
    with pytest.raises(ProtocolError):
        Observation(Status.OK)
    with pytest.raises(ProtocolError):
        Observation(Status.INVALID, time_ms=1.0)
    assert Observation(Status.OK, (1.0,), 1.0).ok


def test_backend_kinds():
    with pytest.raises(ProtocolError):
        BackendDescriptor(kind="gpu")  # pinned by ref tests/test_measure.py:61-62
    with pytest.raises(ProtocolError):
        BackendDescriptor(kind="cuda")  # needs a target
    with pytest.raises(ProtocolError):
        command_backend("echo hi")
    command_backend("echo hi", parameterless=True)


def script_backend(tmp_path, body, template_args="{a}"):
    script = tmp_path / "bench.py"
    script.write_text(textwrap.dedent(body))
    return command_backend(f"{sys.executable} {script} {template_args}")


SPACE = space_from_tune_params("k", {"a": [1, 2]})


def test_counter_drops_warmups(tmp_path):
    counter = tmp_path / "n"
    be = script_backend(tmp_path, f"""
        import pathlib
        p = pathlib.Path({str(counter)!r})
        n = int(p.read_text()) + 1 if p.exists() else 1
        p.write_text(str(n))
        print("TUNE_TIME_MS", n)
    """)
    obs = measure(be, (1,), MeasurementProtocol(warmup_runs=2, benchmark_runs=3), ["a"])
    assert obs.times_ms == (3.0, 4.0, 5.0) and obs.time_ms == 4.0


def test_self_reporting_and_status(tmp_path):
    be = script_backend(tmp_path, """
        for t in (9, 1, 2, 3, 4, 5, 6, 7):
            print("TUNE_TIME_MS", t)
    """)
    obs = measure(be, (1,), MeasurementProtocol(), ["a"])
    assert obs.times_ms == (1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0)
    bad = script_backend(tmp_path, """
        import sys
        print("TUNE_STATUS compile_failed")
        sys.exit(3)
    """)
    assert measure(bad, (1,), MeasurementProtocol(), ["a"]).status is Status.COMPILE_FAILED


def test_timeout_and_garbled(tmp_path):
    slow = script_backend(tmp_path, """
        import time; time.sleep(5)
    """)
    assert measure(slow, (1,), MeasurementProtocol(timeout_ms=300), ["a"]).status is Status.TIMEOUT
    garbled = script_backend(tmp_path, """
        print("TUNE_TIME_MS abc")
    """)
    o = measure(garbled, (1,), MeasurementProtocol(), ["a"])
    assert o.status is Status.RUNTIME_FAILED and "garbled" in o.detail


def test_simulated_and_metric():
    g = bundled_space("gemm")
    c = next(iter(g.enumerate_configs()))
    from paper_2407_11488_b200.paramspace import config_key

    cache = TuningCache("gemm", "d", g.param_names, {config_key(c): Observation(Status.OK, (6.939,), 6.939)})
    be = simulated_backend(cache)
    assert run_config(g, be, MeasurementProtocol(), c).metric_value is None  # verbatim replay
    with pytest.raises(MissingEntry):
        measure(be, list(g.enumerate_configs())[1], MeasurementProtocol())
    assert round(compute_metric(g.metric_source, 6.939, dict(zip(g.param_names, c)))) == 19807
    with pytest.raises(EvaluationError):
        compute_metric(None, 0.0, {})
