"""Cache formats: native v1 round trip and Kernel Tuner interop.

The Kernel-Tuner-format writer is checked against our importer (always)
and against the UNMODIFIED reference importer
(`pkg/src/tunescape/store.py:275-362`) when the reference tree is
present -- the parity bridge of SURVEY §8c.
"""

import json
import random

import pytest

from paper_2407_11488_b200.measure import Observation, Status
from paper_2407_11488_b200.paramspace import bundled_space, config_key
from paper_2407_11488_b200.store import (
    TuningCache,
    dumps_cache,
    import_external_cache,
    loads_cache,
    read_cache,
    write_cache,
    write_kernel_tuner_cache,
)
from paper_2407_11488_b200.errors import CacheFormatError, SpaceMismatch


def sample_cache(space, n=300, seed=0):
    rng = random.Random(seed)
    recs = {}
    for c in list(space.enumerate_configs())[:n]:
        r = rng.random()
        if r < 0.05:
            recs[config_key(c)] = Observation(Status.COMPILE_FAILED, detail="nvrtc: error")
        elif r < 0.1:
            recs[config_key(c)] = Observation(Status.INVALID)
        else:
            ts = tuple(round(rng.uniform(0.01, 5), 6) for _ in range(7))
            t = sum(ts) / 7
            recs[config_key(c)] = Observation(Status.OK, ts, t, space.metric_value(t, c))
    return TuningCache(space.kernel_name, "NVIDIA B200", space.param_names, recs, space.fingerprint())


def test_native_round_trip(tmp_path):
    space = bundled_space("gemm")
    c = sample_cache(space)
    p = write_cache(c, tmp_path / "c.json")
    assert dumps_cache(read_cache(p)) == p.read_text() == dumps_cache(c)
    with pytest.raises(CacheFormatError):
        loads_cache('{"schema_version": 2}')


def test_kernel_tuner_writer_round_trip(tmp_path):
    space = bundled_space("convolution")
    c = sample_cache(space)
    p = write_kernel_tuner_cache(c, tmp_path / "kt.json", space)
    doc = json.loads(p.read_text())
    assert doc["tune_params_keys"] == list(space.param_names)
    back = import_external_cache(p, expected_space=space)
    assert set(back.records) == set(c.records)
    for k, o in c.records.items():
        b = back.records[k]
        assert b.status == o.status
        if o.ok:
            assert b.time_ms == o.time_ms and b.times_ms == o.times_ms


def test_kernel_tuner_cache_imports_into_reference(tmp_path, reference_pkg):
    from tunescape.paramspace import bundled_space as ref_space
    from tunescape.store import import_external_cache as ref_import

    space = bundled_space("hotspot")
    c = sample_cache(space, n=500)
    p = write_kernel_tuner_cache(c, tmp_path / "kt.json", space)
    ref = ref_import(p, expected_space=ref_space("hotspot"))
    assert ref.space_fingerprint == space.fingerprint()
    assert {k: o.status.value for k, o in ref.records.items()} == \
        {k: o.status.value for k, o in c.records.items()}


def test_native_cache_readable_by_reference(tmp_path, reference_pkg):
    from tunescape.store import read_cache as ref_read, dumps_cache as ref_dumps

    space = bundled_space("dedispersion")
    c = sample_cache(space)
    p = write_cache(c, tmp_path / "c.json")
    assert ref_dumps(ref_read(p)) == p.read_text()


def test_outside_space_rejected(tmp_path):
    space = bundled_space("convolution")
    p = tmp_path / "kt.json"
    p.write_text(json.dumps({"tune_params_keys": list(space.param_names),
                             "cache": {"999,1,1,1,0,0,0": {"time": 1.0}}}))
    with pytest.raises(SpaceMismatch):
        import_external_cache(p, expected_space=space)
