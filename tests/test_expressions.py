"""Restriction-language parity with the reference (golden fixtures).

Every case in tests/golden/reference_golden.json was evaluated by the
reference (`pkg/src/tunescape/expressions.py`); we must reproduce the
AST, the static type, every value (by repr, so int/float distinctions
count) and every error class and message.  Mirrors the reference's own
tests (`pkg/tests/test_expressions.py:15-141`).
"""

import random

import numpy as np
import pytest

from paper_2407_11488_b200 import expressions as ex
from paper_2407_11488_b200.errors import EvaluationError, ExpressionSyntaxError, ExpressionTypeError

TYPES = {"a": "int", "b": "int", "c": "int", "mode": "str", "x": "int"}
ENVS = [dict(a=a, b=b, c=c, mode="fast", x=1) for a, b, c in
        [(1, 2, 3), (-4, 3, 2), (7, -2, 0), (0, 5, -3), (12, 4, 1)]]


def test_golden_cases(golden):
    cases = golden["expressions"]
    assert len(cases) > 500
    for rec in cases:
        src = rec["source"]
        if "parse_error" in rec:
            with pytest.raises(ExpressionSyntaxError) as info:
                ex.parse_expression(src)
            assert [type(info.value).__name__, str(info.value)] == rec["parse_error"], src
            continue
        node = ex.parse_expression(src)
        assert repr(node) == rec["ast"], src
        if "type_error" in rec:
            with pytest.raises(ExpressionTypeError) as info:
                ex.check_types(node, TYPES, src)
            assert str(info.value) == rec["type_error"][1], src
            continue
        assert ex.check_types(node, TYPES, src) == rec["type"], src
        for env, (kind, val) in zip(ENVS, rec["values"]):
            if kind == "ok":
                assert repr(ex.evaluate(node, env)) == val, (src, env)
            else:
                # same exception class as the reference (EvaluationError for
                # zero divisors; Python's own errors propagate unchanged)
                with pytest.raises(Exception) as info:
                    ex.evaluate(node, env)
                assert type(info.value).__name__ == val, (src, env)


@pytest.mark.parametrize("source", ["-7 / 2 == -3", "7 / -2 == -3", "-7 % 2 == -1", "7 % -2 == 1",
                                    "2 ^ 10 == 1024", "-2 ^ 2 == -4", "10 / 4 == 2",
                                    "2 * 4096 ^ 3 == 137438953472"])
def test_c_integer_semantics(source):
    assert ex.evaluate(ex.parse_expression(source), {}) is True


def test_error_position():
    with pytest.raises(ExpressionSyntaxError) as info:
        ex.parse_expression("x + $")
    assert info.value.position == 4 and "column 5" in str(info.value)


def test_division_by_zero_raises():
    with pytest.raises(EvaluationError):
        ex.evaluate(ex.parse_expression("x / y"), {"x": 1, "y": 0})


def test_vector_eval_matches_scalar_on_random_expressions(golden):
    """The numpy evaluator is exact wherever it claims to be."""
    rng = np.random.default_rng(0)
    cols = {k: rng.integers(-20, 21, size=400).astype(np.int64) for k in ("a", "b", "c", "x")}
    cols["mode"] = rng.integers(0, 2, size=400)
    ranges = {k: (-20, 20) for k in ("a", "b", "c", "x")}
    ranges["mode"] = ("fast", "slow")
    checked = 0
    for rec in golden["expressions"]:
        if "values" not in rec or rec["type"] != "bool":
            continue
        node = ex.parse_expression(rec["source"])
        try:
            val, err = ex.vector_eval(node, cols, TYPES, ranges)
        except ex.NotVectorizable:
            continue
        names = sorted(ex.variables(node))
        fn = ex.compile_expression(node, names)
        for i in range(400):
            env = {k: (("fast", "slow")[int(cols[k][i])] if k == "mode" else int(cols[k][i]))
                   for k in names}
            try:
                want = fn(*(env[k] for k in names))
                assert err is None or not err[i], rec["source"]
                assert bool(val[i]) == want, (rec["source"], env)
            except ZeroDivisionError:
                assert err is not None and err[i], rec["source"]
        checked += 1
    assert checked > 100


def test_pratt_parser_random_roundtrip():
    rng = random.Random(5)
    for _ in range(200):
        a, b = rng.randint(-9, 9), rng.randint(1, 9)
        node = ex.parse_expression(f"{a} / {b} * {b} + {a} % {b} == {a}")
        assert ex.evaluate(node, {}) is True
