"""The ``tune`` command line (SURVEY §8f row 2; ref ts/cli.py:58-139, :277-283).

Runs on the simulated (replay) backend with the reference's golden
strategy records, so the command's caches and printed results can be
checked against the traces the reference itself produced; plus resume
from a torn observation log and the exit-code contract.
"""

import json
import subprocess
import sys

import pytest
from click.testing import CliRunner

from paper_2407_11488_b200.cli import cli
from paper_2407_11488_b200.paramspace import config_key, parse_space_spec
from paper_2407_11488_b200.store import read_cache, write_cache
from test_strategies import golden_backend


def _setup(golden, tmp_path, which=0):
    rec = golden["strategies"][which]
    s, be = golden_backend(rec)
    spec = tmp_path / "space.spec"
    spec.write_text(rec["text"])
    src = tmp_path / "replay.json"
    write_cache(be.cache, src)
    return rec, s, spec, src


def test_tune_brute_matches_reference_brute_force(golden, tmp_path):
    rec, s, spec, src = _setup(golden, tmp_path)
    out = tmp_path / "out.json"
    kt = tmp_path / "kt.json"
    r = CliRunner().invoke(cli, ["tune", "--space", str(spec), "--backend", f"sim:{src}", "--out", str(out),
                                 "--kt-out", str(kt)])
    assert r.exit_code == 0, r.output
    cache = read_cache(out)
    assert sorted(cache.records) == sorted(s_key for s_key in json.loads(rec["cache_text"])["records"])
    assert cache.metadata == {"strategy": "brute", "seed": "0"}
    want_best = rec["brute_best"]
    if want_best:
        assert f"best config : {want_best}" in r.output
    assert json.loads(kt.read_text())["tune_params_keys"] == list(s.param_names)


def test_tune_random_and_local_traces(golden, tmp_path):
    rec, s, spec, src = _setup(golden, tmp_path)
    checked = 0
    for run in rec["runs"]:
        if run["kind"] not in ("random", "greedy"):
            continue
        out = tmp_path / f"{run['kind']}.json"
        strategy = "random" if run["kind"] == "random" else "local"
        r = CliRunner().invoke(cli, ["tune", "--space", str(spec), "--backend", f"sim:{src}", "--out", str(out),
                                     "--strategy", strategy, "--budget", str(run["budget"]),
                                     "--seed", str(run["seed"])])
        assert r.exit_code == 0, r.output
        assert sorted(read_cache(out).records) == sorted(run["trace"])
        assert f"evaluations : {len(run['trace'])}" in r.output
        if run["best"]:
            assert f"best config : {run['best']}" in r.output
        for note in run["notes"]:
            assert f"note        : {note}" in r.output
        checked += 1
    assert checked >= 2


def test_tune_resume_from_torn_log(golden, tmp_path):
    rec, s, spec, src = _setup(golden, tmp_path)
    log = tmp_path / "obs.jsonl"
    args = ["tune", "--space", str(spec), "--backend", f"sim:{src}", "--resume", str(log), "--chunk", "3"]
    r = CliRunner().invoke(cli, args + ["--out", str(tmp_path / "a.json")])
    assert r.exit_code == 0, r.output
    lines = log.read_text().splitlines()
    n = s.space_size()
    assert len(lines) == n + 1 and '"header"' in lines[0]  # space fingerprint + protocol
    # keep a third of the log plus a torn half line, as a crash would
    keep = lines[: n // 3]
    log.write_text("\n".join(keep) + "\n" + lines[n // 3][: 10])
    r = CliRunner().invoke(cli, args + ["--out", str(tmp_path / "b.json")])
    assert r.exit_code == 0, r.output
    good = [json.loads(x) for x in log.read_text().splitlines() if x.startswith("{") and x.endswith("}")]
    good = [d for d in good if "key" in d]
    assert sorted(d["key"] for d in good) == sorted(json.loads(x)["key"] for x in lines[1:])
    a, b = read_cache(tmp_path / "a.json"), read_cache(tmp_path / "b.json")
    assert a.records == b.records
    assert sorted(a.records) == sorted(config_key(c) for c in s.enumerate_configs())


def test_resume_refuses_a_log_of_another_protocol(golden, tmp_path):
    """Observations measured under another protocol (or space) are not reused."""
    rec, s, spec, src = _setup(golden, tmp_path)
    log = tmp_path / "obs.jsonl"
    base = ["tune", "--space", str(spec), "--backend", f"sim:{src}", "--resume", str(log)]
    assert CliRunner().invoke(cli, base + ["--out", str(tmp_path / "a.json")]).exit_code == 0
    r = CliRunner().invoke(cli, base + ["--runs", "3", "--out", str(tmp_path / "b.json")])
    assert r.exit_code != 0 and "another protocol" in str(r.exception)


def test_exit_codes(golden, tmp_path):
    rec, s, spec, src = _setup(golden, tmp_path)
    # domain error -> "error: <Type>: ..." and exit 1 (ref ts/cli.py:277-283)
    p = subprocess.run([sys.executable, "-m", "paper_2407_11488_b200", "tune", "--space",
                        str(tmp_path / "missing.spec"), "--backend", f"sim:{src}", "--out",
                        str(tmp_path / "x.json")], capture_output=True, text=True, timeout=120)
    assert p.returncode == 1 and p.stderr.startswith("error: SpecValidationError"), p.stderr
    # usage errors -> exit 2
    r = CliRunner().invoke(cli, ["tune", "--space", str(spec), "--backend", "gpu:x", "--out", "y.json"])
    assert r.exit_code == 2
    r = CliRunner().invoke(cli, ["tune", "--space", str(spec), "--backend", f"sim:{src}", "--out", "y.json",
                                 "--devices", "2"])
    assert r.exit_code == 2
    assert parse_space_spec(rec["text"]).space_size() == s.space_size()


@pytest.mark.gpu
def test_tune_cuda_backend(tmp_path):
    """``--backend cuda:<kernel>`` end to end on the GPU: random search over
    the convolution space, then a resumed brute-force slice of the same log."""
    out = tmp_path / "conv.json"
    r = CliRunner().invoke(cli, ["tune", "--space", "convolution", "--backend", "cuda:convolution",
                                 "--strategy", "random", "--budget", "6", "--seed", "1", "--out", str(out),
                                 "--kt-out", str(tmp_path / "conv_kt.json")])
    assert r.exit_code == 0, (r.output, r.exception)
    cache = read_cache(out)
    assert len(cache.records) == 6
    assert "B200" in cache.device_name
    assert any(o.ok for o in cache.records.values())
    assert "best config : " in r.output
    r = CliRunner().invoke(cli, ["tune", "--space", "dedispersion", "--backend", "cuda:convolution",
                                 "--out", str(tmp_path / "bad.json")])
    assert r.exit_code != 0 and "does not match" in str(r.exception)


def test_resume_counts_every_rank_log(golden, tmp_path):
    """A restarted sweep treats observations in ANY earlier log (one per rank
    of a multi-GPU run) as done: nothing is measured twice."""
    from paper_2407_11488_b200.multigpu import sharded_sweep
    from paper_2407_11488_b200.measure import MeasurementProtocol
    from paper_2407_11488_b200.store import ResultLog

    rec, s, spec, src = _setup(golden, tmp_path)
    be = golden_backend(rec)[1]
    configs = list(s.enumerate_configs())
    # an earlier 2-rank run logged disjoint halves under <log>.rank0/.rank1
    base = tmp_path / "obs.jsonl"
    for r, part in enumerate((configs[::2], configs[1::2])):
        lg = ResultLog(f"{base}.rank{r}")
        for c in part:
            lg.append(",".join(map(str, c)), be.cache.records[",".join(map(str, c))])
        lg.close()
    calls = []
    be2 = golden_backend(rec)[1]
    orig = be2.cache.records.get

    class Spy(dict):
        def get(self, k, d=None):
            calls.append(k)
            return orig(k, d)

    be2.cache.records = Spy(be2.cache.records)
    trace, _ = sharded_sweep(s, configs, be2, MeasurementProtocol(), 3, log_path=f"{base}.rank0",
                             resume_from=[str(base), f"{base}.rank0", f"{base}.rank1"])
    assert [c for c, _ in trace] == configs
    assert calls == []  # everything came from the logs


@pytest.mark.gpu
def test_tune_sharded_over_ranks_on_the_gpu(tmp_path):
    """``--devices 2``: the command re-launches itself as two torchrun ranks
    (on a one-GPU host both share it -- the functional path of the sharded
    sweep: TCPStore chunk queue, gloo gather, merge by draw order); the
    random search's pre-drawn sequence gives exactly the single-process
    run's configurations, every one measured and verified on the device."""
    args = ["--space", "convolution", "--backend", "cuda:convolution", "--strategy", "random",
            "--budget", "8", "--seed", "3"]
    one, two = tmp_path / "one.json", tmp_path / "two.json"
    base = [sys.executable, "-m", "paper_2407_11488_b200", "tune"]
    r1 = subprocess.run(base + args + ["--out", str(one)], capture_output=True, text=True, timeout=900)
    assert r1.returncode == 0, r1.stderr[-2000:]
    r2 = subprocess.run(base + args + ["--devices", "2", "--out", str(two)], capture_output=True, text=True,
                        timeout=900)
    assert r2.returncode == 0, r2.stderr[-2000:]
    c1, c2 = read_cache(one), read_cache(two)
    assert list(c1.records) == list(c2.records) and len(c2.records) == 8
    assert all(o.ok for o in c2.records.values())
    assert [o.status for o in c1.records.values()] == [o.status for o in c2.records.values()]
