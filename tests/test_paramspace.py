"""Search-space parity with the reference.

Counts, enumeration order (SHA-256 of ordered keys), canonical text and
fingerprints of the four bundled spaces, neighbourhoods, and random
spaces against the reference's Cartesian-filter oracle pattern
(`pkg/tests/conftest.py:126-138`).
"""

import hashlib
import random
from itertools import product

import numpy as np
import pytest

from paper_2407_11488_b200 import expressions as ex
from paper_2407_11488_b200.errors import EvaluationError, SpecSyntaxError, SpecValidationError
from paper_2407_11488_b200.paramspace import (
    ConstraintExpr,
    ParameterDef,
    SearchSpaceSpec,
    bundled_space,
    config_key,
    parse_space_spec,
    space_from_tune_params,
)

APPENDIX_A = {
    "convolution": (10240, 4362, "9242338fb7d801e1dfc1985408999919d673b6edea5b3e1944557d28c99a1227"),
    "hotspot": (4440000, 105412, "091082499b7484354e4c8fa3cd93b3cfa476e7537b8edabc8a81425bf6eac806"),
    "dedispersion": (22272, 11130, "031166ce971c03471898116a3a83220762abcc9753b63d1d416e232cd253ddfb"),
    "gemm": (663552, 116928, "c89db77cbace1ce03c49e4d918a90ebc00759a7cb7744f24777763c3b93d724d"),
}


def digest(configs) -> str:
    h = hashlib.sha256()
    for c in configs:
        h.update((config_key(c) + "\n").encode())
    return h.hexdigest()


@pytest.mark.parametrize("name", sorted(APPENDIX_A))
def test_bundled_space_matches_reference(name, golden):
    s = bundled_space(name)
    ref = golden["spaces"][name]
    cart, valid, dig = APPENDIX_A[name]
    configs = list(s.enumerate_configs())
    assert s.cartesian_size == cart == ref["cartesian"]
    assert len(configs) == valid == ref["valid"] == s.space_size()
    assert digest(configs) == dig == ref["digest"]
    assert config_key(configs[0]) == ref["first"] and config_key(configs[-1]) == ref["last"]
    assert s.to_text() == ref["text"]
    assert s.fingerprint() == ref["fingerprint"]
    for key, nbrs in ref["neighbors"].items():
        assert [config_key(n) for n in s.neighbors(s.config_from_key(key))] == nbrs
    for key, nbrs in ref["neighbors_adjacent"].items():
        assert [config_key(n) for n in s.neighbors(s.config_from_key(key), "adjacent")] == nbrs


def test_hotspot_per_t_counts(golden):
    s = bundled_space("hotspot")
    idx = s.valid_indices()
    t_vals = np.array([c[4] for c in s.configs_at(idx)])
    counts = {str(t): int((t_vals == t).sum()) for t in range(1, 11)}
    assert counts == {str(k): v for k, v in golden["spaces"]["hotspot"]["per_temporal_tiling_factor"].items()}
    assert [counts[str(t)] for t in range(1, 11)] == [6085, 10738, 9730, 13371, 8230, 15260, 7244,
                                                      13508, 9462, 11784]


def test_hotspot_smem_over_48k():
    s = bundled_space("hotspot")
    n = 0
    for c in s.enumerate_configs():
        bx, by, tx, ty, t, _, shp = c
        if (2 + shp) * (bx * tx + 2 * t) * (by * ty + 2 * t) * 4 > 48 * 1024:
            n += 1
    assert n == 22428


_POOL = ("{a} * {b} <= {cap}", "{a} % {b} == 0", "{a} <= {b}", "{a} + {b} >= {low}",
         "{a} == {v} || {b} != {v}", "({a} - {b}) / 2 != 1", "!({a} == {v})")


def random_space(rng):
    params = {}
    for i in range(rng.randint(2, 5)):
        start, step = rng.randint(-3, 4), rng.randint(1, 4)
        params[f"p{i}"] = [start + step * j for j in range(rng.randint(2, 7))]
    names = list(params)
    cons = []
    for _ in range(rng.randint(0, 3)):
        a, b = rng.sample(names, 2)
        cons.append(rng.choice(_POOL).format(a=a, b=b, cap=rng.choice([16, 64, 256]),
                                             low=rng.randint(2, 8), v=rng.choice(params[a])))
    return space_from_tune_params("r", params, cons)


def oracle_valid(space):
    names = sorted(space.param_names)
    order = [space.param_names.index(n) for n in names]
    checks = [ex.compile_expression(c.ast, names) for c in space.constraints]
    out = []
    for combo in product(*(p.values for p in space.parameters)):
        re = [combo[i] for i in order]
        try:
            if all(fn(*re) for fn in checks):
                out.append(combo)
        except ZeroDivisionError:
            return None
    return out


def test_random_spaces_vs_cartesian_oracle():
    rng = random.Random(42)
    for _ in range(200):
        s = random_space(rng)
        want = oracle_valid(s)
        if want is None:
            continue
        assert list(s.enumerate_configs()) == want
        # scalar path agrees with the vectorised path
        assert list(s._filter_scalar()) == want


def test_golden_random_spaces(golden):
    for rec in golden["strategies"]:
        s = parse_space_spec(rec["text"])
        assert [config_key(c) for c in s.enumerate_configs()] == rec["valid"]


def test_zero_division_surfaces_config():
    s = space_from_tune_params("z", {"a": [1, 2], "b": [0, 1]}, ["a / b >= 1"])
    with pytest.raises(EvaluationError, match=r"\(1,0\)"):
        list(s.enumerate_configs())
    # short-circuit: the divisor is never reached when the guard fails
    s2 = space_from_tune_params("z", {"a": [1, 2], "b": [0, 1]}, ["b != 0 && a / b >= 1"])
    assert list(s2.enumerate_configs()) == [(1, 1), (2, 1)]


def test_large_power_falls_back_exactly():
    s = space_from_tune_params("p", {"a": [2, 3], "b": [40, 70]}, ["a ^ b > 2 ^ 60"])
    assert list(s.enumerate_configs()) == [(2, 70), (3, 40), (3, 70)]


def test_string_parameters():
    s = space_from_tune_params("s", {"mode": ["fast", "slow"], "n": [1, 2, 3]},
                               ["mode == 'fast' || n > 1"])
    assert list(s.enumerate_configs()) == [("fast", 1), ("fast", 2), ("fast", 3), ("slow", 2), ("slow", 3)]


def test_callable_restriction_kernel_tuner_style():
    s = space_from_tune_params("k", {"x": [1, 2, 4], "y": [1, 2]},
                               [lambda p: p["x"] * p["y"] <= 4, "x >= 2"])
    assert list(s.enumerate_configs()) == [(2, 1), (2, 2), (4, 1)]


def test_spec_errors():
    with pytest.raises(SpecSyntaxError):
        parse_space_spec("kernel: k\nkernel: j\nparams:\n  a: [1]\n")
    with pytest.raises(SpecValidationError):
        parse_space_spec("kernel: k\nparams:\n  a: [1.5]\n")
    with pytest.raises(SpecValidationError):
        parse_space_spec("kernel: k\nbogus: 1\nparams:\n  a: [1]\n")


def test_flat_index_roundtrip():
    s = bundled_space("gemm")
    idx = s.valid_indices()
    for flat in idx[:: max(1, len(idx) // 50)]:
        c = s.config_at(int(flat))
        assert s.flat_index(c) == flat and s.is_valid(c)


def test_metric_known_answers(golden):
    g = bundled_space("gemm")
    c = next(iter(g.enumerate_configs()))
    assert g.metric_value(6.939, c) == pytest.approx(golden["metric"]["gemm_6.939"], rel=0, abs=0)
    assert round(g.metric_value(6.939, c)) == 19807
    conv = bundled_space("convolution")
    assert conv.metric_value(1.0, next(iter(conv.enumerate_configs()))) == golden["metric"]["conv_1.0"]
