"""Caches produced on the B200 by a full brute-force sweep (tools/full_sweep.py).

The committed convolution cache covers all 4,362 valid configurations of the
reference space, measured with the in-process ``cuda`` backend.  It must read
back through our own reader and -- the parity bridge of SURVEY §8c -- import
into the UNMODIFIED reference with ``expected_space`` (no SpaceMismatch) and
yield a complete landscape (the reference's ``build_ffg`` raises
IncompleteCache otherwise).
"""

import gzip
import json
from pathlib import Path

import pytest

from paper_2407_11488_b200.paramspace import bundled_space, config_key
from paper_2407_11488_b200.store import import_external_cache, loads_cache

CACHES = Path(__file__).resolve().parents[1] / "profiles" / "round1" / "caches"


def _unzip(name: str, tmp_path: Path) -> Path:
    p = tmp_path / name
    p.write_bytes(gzip.decompress((CACHES / (name + ".gz")).read_bytes()))
    return p


def test_gpu_convolution_cache_is_complete(tmp_path):
    space = bundled_space("convolution")
    keys = {config_key(c) for c in space.enumerate_configs()}
    native = loads_cache(_unzip("convolution.tunescape.json", tmp_path).read_text())
    assert set(native.records) == keys and len(keys) == 4362
    assert all(o.ok and o.time_ms > 0 and len(o.times_ms) == 7 for o in native.records.values())
    kt = import_external_cache(_unzip("convolution.kerneltuner.json", tmp_path), expected_space=space)
    assert set(kt.records) == keys
    summary = json.loads((CACHES / "convolution.summary.json").read_text())
    best = min(native.records.items(), key=lambda kv: kv[1].time_ms)
    assert best[0] == ",".join(map(str, summary["best"]))


def test_gpu_convolution_cache_imports_into_reference(tmp_path, reference_pkg):
    from tunescape.landscape import build_ffg
    from tunescape.paramspace import bundled_space as ref_space
    from tunescape.store import import_external_cache as ref_import

    rs = ref_space("convolution")
    ref = ref_import(_unzip("convolution.kerneltuner.json", tmp_path), expected_space=rs)
    assert len(ref.records) == 4362
    assert ref.space_fingerprint == bundled_space("convolution").fingerprint()
    ffg = build_ffg(ref, rs)  # raises IncompleteCache unless every valid configuration is present
    assert ffg is not None


def test_gpu_dedispersion_cache_is_complete(tmp_path):
    """The whole dedispersion space (11,130 configurations) swept on a B200
    through the tune command line (all verified bit-exact on the device)."""
    space = bundled_space("dedispersion")
    keys = {config_key(c) for c in space.enumerate_configs()}
    native = loads_cache(_unzip("dedispersion.tunescape.json", tmp_path).read_text())
    assert set(native.records) == keys and len(keys) == 11130
    assert all(o.ok and o.time_ms > 0 and len(o.times_ms) == 7 for o in native.records.values())
    kt = import_external_cache(_unzip("dedispersion.kerneltuner.json", tmp_path), expected_space=space)
    assert set(kt.records) == keys
    summary = json.loads((CACHES / "dedispersion.summary.json").read_text())
    best = min(native.records.items(), key=lambda kv: kv[1].time_ms)
    assert best[0] == ",".join(map(str, summary["best"]))


def test_gpu_dedispersion_cache_imports_into_reference(tmp_path, reference_pkg):
    from tunescape.landscape import build_ffg
    from tunescape.paramspace import bundled_space as ref_space
    from tunescape.store import import_external_cache as ref_import

    rs = ref_space("dedispersion")
    ref = ref_import(_unzip("dedispersion.kerneltuner.json", tmp_path), expected_space=rs)
    assert len(ref.records) == 11130
    assert build_ffg(ref, rs) is not None  # complete landscape


# ---- round 2: all four spaces swept with the final kernels -----------------
CACHES2 = Path(__file__).resolve().parents[1] / "profiles" / "round2" / "caches"
FULL2 = {"hotspot": 105412, "gemm": 116928, "convolution": 4362, "dedispersion": 11130}


def _unzip2(name: str, tmp_path: Path) -> Path:
    p = tmp_path / name
    p.write_bytes(gzip.decompress((CACHES2 / (name + ".gz")).read_bytes()))
    return p


def _swept(problem: str) -> bool:
    return (CACHES2 / f"{problem}.tunescape.json.gz").exists()


@pytest.mark.parametrize("problem", sorted(FULL2))
def test_round2_full_space_cache(problem, tmp_path, reference_pkg):
    """A whole reference space swept on a B200 through the tune command line
    (every configuration verified on the device): complete in our format,
    the Kernel-Tuner export imports into the UNMODIFIED reference with
    ``expected_space`` and its ``build_ffg`` (IncompleteCache otherwise)
    builds the complete landscape; the summary's best is the cache's best."""
    if not _swept(problem):
        pytest.skip(f"{problem}: full-space sweep not committed")
    from tunescape.landscape import build_ffg
    from tunescape.paramspace import bundled_space as ref_space
    from tunescape.store import import_external_cache as ref_import

    space = bundled_space(problem)
    keys = {config_key(c) for c in space.enumerate_configs()}
    assert len(keys) == FULL2[problem]
    native = loads_cache(_unzip2(f"{problem}.tunescape.json", tmp_path).read_text())
    assert set(native.records) == keys
    ok = native.ok_records()
    assert all(o.time_ms > 0 and len(o.times_ms) == 7 for o in ok.values())
    summary = json.loads((CACHES2 / f"{problem}.summary.json").read_text())
    best = min(ok.items(), key=lambda kv: kv[1].time_ms)
    assert best[0] == ",".join(map(str, summary["best"])) and summary["ok"] == len(ok)
    rs = ref_space(problem)
    ref = ref_import(_unzip2(f"{problem}.kerneltuner.json", tmp_path), expected_space=rs)
    assert len(ref.records) == len(keys)
    assert build_ffg(ref, rs) is not None  # complete landscape
