"""The restriction / metric expression language.

Behavioural contract (reference `pkg/src/tunescape/expressions.py:1-28`):

* precedence, loosest first: ``||``/``or``, ``&&``/``and``, prefix
  ``!``/``not``, one *non-chaining* comparison, ``+ -``, ``* / %``,
  prefix ``-``, right-associative ``^`` whose exponent may carry a
  prefix minus (``-2^2 == -4``, ``2^-1 == 0.5``);
* integers are exact; ``/`` truncates toward zero and ``%`` keeps the
  dividend's sign (C semantics, ref :295-311); any float operand makes
  the operation a float; a zero divisor raises :class:`EvaluationError`
  at the evaluation site;
* strings only compare with ``==``/``!=``; boolean operators need
  boolean operands (static check, ref :230-292).

Implementation here is independent of the reference: a table-driven
Pratt parser, a type inferencer over the same node set, a Python code
generator for the scalar path, and -- new for the B200 build -- a
numpy evaluator (:func:`vector_eval`) that filters millions of
Cartesian points per call while keeping C integer semantics bit-exact
(guarded by an interval analysis that falls back to the scalar path
whenever int64 could overflow).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Mapping, Sequence, Union

import numpy as np

from .errors import EvaluationError, ExpressionSyntaxError, ExpressionTypeError

Scalar = Union[int, float, str]

# --------------------------------------------------------------------------
# AST.  The class and field names are part of the golden contract: the
# fixtures record ``repr(parse_expression(src))`` as the reference prints
# it (``Binary(op='+', left=Num(value=1), right=Var(name='x'))``), so the
# five node kinds keep exactly these names and field orders.  Each node
# knows its children, which lets every traversal below be one generic
# post-order walk instead of an isinstance ladder per pass.


class _Node:
    __slots__ = ()

    def children(self) -> tuple:
        return ()


@dataclass(frozen=True, slots=True)
class Num(_Node):
    value: int | float


@dataclass(frozen=True, slots=True)
class Str(_Node):
    value: str


@dataclass(frozen=True, slots=True)
class Var(_Node):
    name: str


@dataclass(frozen=True, slots=True)
class Unary(_Node):
    op: str  # '-' or '!'
    operand: "Node"

    def children(self) -> tuple:
        return (self.operand,)


@dataclass(frozen=True, slots=True)
class Binary(_Node):
    op: str
    left: "Node"
    right: "Node"

    def children(self) -> tuple:
        return (self.left, self.right)


Node = Union[Num, Str, Var, Unary, Binary]

COMPARISONS = frozenset({"==", "!=", "<", "<=", ">", ">="})
ARITHMETIC = frozenset({"+", "-", "*", "/", "%", "^"})
LOGICAL = frozenset({"&&", "||"})


def postorder(node: Node):
    """Nodes of ``node`` children-first, left to right (iterative)."""
    stack = [(node, False)]
    while stack:
        n, expanded = stack.pop()
        if expanded:
            yield n
            continue
        stack.append((n, True))
        stack.extend((c, False) for c in reversed(n.children()))


# --------------------------------------------------------------------------
# Lexer: a hand-written scanner.  Token classes and their precedence follow
# the grammar of ``ts/expressions.py:1-28``: a number is a float when it has
# a '.' mantissa or a complete exponent (``1e5``, ``1.``, ``.5``), else an
# integer (``1e`` is the integer 1 followed by the name ``e``); names are
# ASCII identifiers; strings are single- or double-quoted with no escapes;
# ``and``/``or``/``not`` are spellings of ``&&``/``||``/``!``.

_WORD_OPS = {"and": "&&", "or": "||", "not": "!"}
_TWO_CHAR_OPS = frozenset({"||", "&&", "==", "!=", "<=", ">="})
_ONE_CHAR_OPS = frozenset("-+*/%^<>!()")
_NAME_START = frozenset("ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz_")
_NAME_CHARS = _NAME_START | frozenset("0123456789")


@dataclass(frozen=True)
class Token:
    kind: str  # int | float | name | string | op | end
    text: str
    pos: int


def _digits_end(s: str, i: int) -> int:
    while i < len(s) and s[i].isdecimal():
        i += 1
    return i


def _exponent_end(s: str, i: int) -> int:
    """End of a complete exponent ``[eE][+-]?digits`` at ``i``, else ``i``."""
    if i < len(s) and s[i] in "eE":
        j = i + 1
        if j < len(s) and s[j] in "+-":
            j += 1
        k = _digits_end(s, j)
        if k > j:
            return k
    return i


def _scan_number(s: str, i: int) -> tuple:
    """(kind, end) of the number starting at ``i`` (a digit or '.digit')."""
    j = _digits_end(s, i)
    if j < len(s) and s[j] == ".":
        if j > i or _digits_end(s, j + 1) > j + 1:  # 'd.' / 'd.d' / '.d'
            return "float", _exponent_end(s, _digits_end(s, j + 1))
    k = _exponent_end(s, j)
    return ("float", k) if k > j else ("int", j)


def tokenize(source: str) -> list[Token]:
    out: list[Token] = []
    i, n = 0, len(source)
    while i < n:
        ch = source[i]
        if ch.isspace():
            i += 1
            continue
        if ch.isdecimal() or (ch == "." and i + 1 < n and source[i + 1].isdecimal()):
            kind, end = _scan_number(source, i)
        elif ch in _NAME_START:
            end = i + 1
            while end < n and source[end] in _NAME_CHARS:
                end += 1
            kind = "name"
        elif ch in "'\"" and source.find(ch, i + 1) >= 0:
            kind, end = "string", source.find(ch, i + 1) + 1
        elif source[i:i + 2] in _TWO_CHAR_OPS:
            kind, end = "op", i + 2
        elif ch in _ONE_CHAR_OPS:
            kind, end = "op", i + 1
        else:
            raise ExpressionSyntaxError(f"unexpected character {ch!r}", source, i)
        text = source[i:end]
        if kind == "name" and text in _WORD_OPS:
            kind, text = "op", _WORD_OPS[text]
        out.append(Token(kind, text, i))
        i = end
    out.append(Token("end", "", n))
    return out


# --------------------------------------------------------------------------
# Pratt parser.  Left binding powers of infix operators:
_INFIX_BP = {"||": 10, "&&": 20, "+": 40, "-": 40, "*": 50, "/": 50, "%": 50, "^": 70}
for _op in COMPARISONS:
    _INFIX_BP[_op] = 30
_NOT_OPERAND_BP = 25  # '!' covers a whole comparison but not && / ||
_NEG_OPERAND_BP = 60  # '-' covers a power but not * / %
_POW_RHS_BP = 70  # right-assoc: rhs may contain another '^' (and a '-')


class _Pratt:
    def __init__(self, source: str):
        self.src = source
        self.toks = tokenize(source)
        self.k = 0

    def peek(self) -> Token:
        return self.toks[self.k]

    def take(self) -> Token:
        t = self.toks[self.k]
        self.k += 1
        return t

    def error(self, expected: str):
        t = self.peek()
        found = "end of expression" if t.kind == "end" else repr(t.text)
        raise ExpressionSyntaxError(f"expected {expected}, found {found}", self.src, t.pos)

    def run(self) -> Node:
        node = self.expr(0)
        if self.peek().kind != "end":
            self.error("end of expression")
        return node

    def prefix(self) -> Node:
        t = self.peek()
        if t.kind == "op" and t.text == "!":
            self.take()
            return Unary("!", self.expr(_NOT_OPERAND_BP))
        if t.kind == "op" and t.text == "-":
            self.take()
            return Unary("-", self.expr(_NEG_OPERAND_BP))
        if t.kind == "int":
            self.take()
            return Num(int(t.text))
        if t.kind == "float":
            self.take()
            return Num(float(t.text))
        if t.kind == "string":
            self.take()
            return Str(t.text[1:-1])
        if t.kind == "name":
            self.take()
            return Var(t.text)
        if t.kind == "op" and t.text == "(":
            self.take()
            inner = self.expr(0)
            if not (self.peek().kind == "op" and self.peek().text == ")"):
                self.error("')'")
            self.take()
            return inner
        self.error("a value, identifier or '('")

    def expr(self, min_bp: int) -> Node:
        left = self.prefix()
        compared = False
        powered = False
        while True:
            t = self.peek()
            if t.kind != "op" or t.text not in _INFIX_BP:
                return left
            op = t.text
            bp = _INFIX_BP[op]
            if bp < min_bp or (bp == min_bp and op != "^"):
                return left
            if op in COMPARISONS and compared:
                return left  # comparisons do not chain; caller reports it
            if op == "^" and powered:
                return left
            self.take()
            if op == "^":
                # exponent: a full prefix-unary, itself possibly a power
                right = self.expr(_POW_RHS_BP)
                powered = True
            else:
                right = self.expr(bp + 1)
            left = Binary(op, left, right)
            if op in COMPARISONS:
                compared = True


def parse_expression(source: str) -> Node:
    """Parse ``source`` into an AST (raises :class:`ExpressionSyntaxError`)."""
    return _Pratt(source).run()


def variables(node: Node) -> set[str]:
    """Identifiers referenced by ``node``."""
    return {n.name for n in postorder(node) if isinstance(n, Var)}


# --------------------------------------------------------------------------
# Static types.  Types are inferred children-first over ``postorder``; each
# operator class has one rule mapping its operand types to a result type or
# to a diagnostic.  Because children are typed before their parent, the
# diagnostic reported is the one of the left-most, inner-most offending
# node -- the order the reference's recursive checker reports in, which the
# golden fixtures pin together with the message texts.

_NUMERIC = ("int", "float")


def _rule_not(op, a):
    return "bool" if a == "bool" else (None, "'!' needs a boolean operand")


def _rule_neg(op, a):
    return a if a in _NUMERIC else (None, "unary '-' needs a number")


def _rule_logical(op, a, b):
    if a == b == "bool":
        return "bool"
    return None, f"'{op}' needs boolean operands"


def _rule_compare(op, a, b):
    if "bool" in (a, b):
        return None, f"cannot compare boolean results with '{op}'"
    if (a == "str") != (b == "str"):
        return None, "cannot compare string and number"
    if a == "str" and op not in ("==", "!="):
        return None, "strings support only '==' and '!='"
    return "bool"


def _rule_arith(op, a, b):
    if a not in _NUMERIC or b not in _NUMERIC:
        return None, f"'{op}' needs numeric operands"
    return "float" if "float" in (a, b) else "int"


_UNARY_RULES = {"!": _rule_not, "-": _rule_neg}
_BINARY_RULES = {**{op: _rule_logical for op in LOGICAL},
                 **{op: _rule_compare for op in COMPARISONS},
                 **{op: _rule_arith for op in ARITHMETIC}}


def check_types(node: Node, var_types: Mapping[str, str], source: str = "") -> str:
    """Return 'int' | 'float' | 'str' | 'bool' or raise ExpressionTypeError."""
    where = f" in {source!r}" if source else ""
    typed: dict = {}
    for n in postorder(node):
        if isinstance(n, Num):
            t = "float" if isinstance(n.value, float) else "int"
        elif isinstance(n, Str):
            t = "str"
        elif isinstance(n, Var):
            t = var_types.get(n.name)
            if t is None:
                raise ExpressionTypeError(f"unknown identifier '{n.name}'{where}")
        else:
            rule = (_UNARY_RULES if isinstance(n, Unary) else _BINARY_RULES)[n.op]
            t = rule(n.op, *(typed[id(c)] for c in n.children()))
            if isinstance(t, tuple):
                raise ExpressionTypeError(t[1] + where)
        typed[id(n)] = t
    return typed[id(node)]


# --------------------------------------------------------------------------
# Scalar semantics


def c_div(a, b):
    """C division: truncating on integers, true division on floats."""
    if b == 0:
        raise ZeroDivisionError("division by zero")
    if type(a) is int and type(b) is int:
        q = abs(a) // abs(b)
        return q if (a < 0) == (b < 0) else -q
    return a / b


def c_mod(a, b):
    """C remainder: sign of the dividend; fmod on floats."""
    if b == 0:
        raise ZeroDivisionError("modulo by zero")
    if type(a) is int and type(b) is int:
        return a - c_div(a, b) * b
    return math.fmod(a, b)


_PY_INFIX = {"&&": "and", "||": "or", "^": "**"}


def _py(n: Node, names: Mapping[str, str]) -> str:
    if isinstance(n, Num) or isinstance(n, Str):
        return repr(n.value)
    if isinstance(n, Var):
        return names[n.name]
    if isinstance(n, Unary):
        inner = _py(n.operand, names)
        return f"(not {inner})" if n.op == "!" else f"(-{inner})"
    a, b = _py(n.left, names), _py(n.right, names)
    if n.op == "/":
        return f"_div({a}, {b})"
    if n.op == "%":
        return f"_mod({a}, {b})"
    return f"({a} {_PY_INFIX.get(n.op, n.op)} {b})"


def compile_expression(node: Node, names: Sequence[str]) -> Callable[..., Scalar]:
    """Positional Python callable over ``names`` (one argument per name).

    Only ASTs from :func:`parse_expression` are rendered, so no foreign
    text reaches ``eval``.
    """
    slots = {name: f"a{i}" for i, name in enumerate(names)}
    params = ", ".join(slots[n] for n in names)
    code = f"lambda {params}: {_py(node, slots)}"
    return eval(code, {"__builtins__": {}, "_div": c_div, "_mod": c_mod})


def evaluate(node: Node, env: Mapping[str, Scalar]):
    """One-off evaluation against a mapping (ZeroDivision -> EvaluationError)."""
    names = sorted(variables(node))
    fn = compile_expression(node, names)
    try:
        return fn(*(env[k] for k in names))
    except ZeroDivisionError as e:
        raise EvaluationError(str(e)) from None


# --------------------------------------------------------------------------
# Vectorised evaluation (new): numpy over many configurations at once.

_I64_SAFE = 2**62


class NotVectorizable(Exception):
    """The expression cannot be evaluated exactly with numpy; use scalar."""


def _bounds(n: Node, ranges: Mapping[str, tuple]) -> tuple:
    """Conservative (lo, hi) for numeric nodes; raises NotVectorizable."""
    if isinstance(n, Num):
        return (n.value, n.value)
    if isinstance(n, Var):
        if n.name not in ranges:
            raise NotVectorizable(f"no value range for {n.name!r}")
        return ranges[n.name]
    if isinstance(n, Unary):
        lo, hi = _bounds(n.operand, ranges)
        return (-hi, -lo)
    lo1, hi1 = _bounds(n.left, ranges)
    lo2, hi2 = _bounds(n.right, ranges)
    op = n.op
    if op == "+":
        return (lo1 + lo2, hi1 + hi2)
    if op == "-":
        return (lo1 - hi2, hi1 - lo2)
    if op == "*":
        c = (lo1 * lo2, lo1 * hi2, hi1 * lo2, hi1 * hi2)
        return (min(c), max(c))
    if op in ("/", "%"):
        m = max(abs(lo1), abs(hi1))
        return (-m, m)  # |a/b| <= |a| for |b| >= 1; |a%b| <= |a|
    if op == "^":
        if lo2 < 0:
            raise NotVectorizable("negative exponent")
        m = max(abs(lo1), abs(hi1))
        if m > 1 and hi2 * math.log2(max(m, 2)) > 62:
            raise NotVectorizable("power may overflow int64")
        big = m ** int(hi2) if hi2 >= 0 else 1
        return (-big, big)
    raise NotVectorizable(op)


def _numeric_nodes(n: Node):
    """Yield maximal arithmetic sub-trees (to bound-check them)."""
    if isinstance(n, Binary) and (n.op in LOGICAL or n.op in COMPARISONS):
        yield from _numeric_nodes(n.left)
        yield from _numeric_nodes(n.right)
    elif isinstance(n, Unary) and n.op == "!":
        yield from _numeric_nodes(n.operand)
    elif not isinstance(n, Str):
        yield n


def vector_eval(node: Node, cols: Mapping[str, np.ndarray], var_types: Mapping[str, str],
                ranges: Mapping[str, tuple]):
    """Evaluate ``node`` over parallel columns.

    ``cols[name]`` is an int64 array for int parameters or an int array
    of *string codes* for str parameters (``var_types`` says which, and
    ``ranges[name]`` for str params is the code->string tuple).
    Returns ``(values, err)`` where ``err`` marks rows whose scalar
    evaluation would have raised (respecting && / || short-circuit);
    raises :class:`NotVectorizable` when exactness cannot be guaranteed.
    """
    num_ranges = {k: v for k, v in ranges.items() if var_types.get(k) != "str"}
    strings_of = {k: v for k, v in ranges.items() if var_types.get(k) == "str"}
    for sub in _numeric_nodes(node):
        if _contains_str(sub) or _is_str_var(sub, var_types):
            continue
        has_float = _contains_float(sub)
        if has_float and _contains_pow(sub):
            raise NotVectorizable("float power (Python may return complex)")
        lo, hi = _bounds(sub, num_ranges)
        limit = 2 ** 53 if has_float else _I64_SAFE
        if max(abs(lo), abs(hi)) >= limit:
            raise NotVectorizable("value range exceeds exact numpy arithmetic")
    nrows = len(next(iter(cols.values()))) if cols else 1

    def ev(n: Node):
        if isinstance(n, Num):
            return n.value, None
        if isinstance(n, Str):
            return n, None  # resolved by the comparison
        if isinstance(n, Var):
            return cols[n.name], None
        if isinstance(n, Unary):
            v, e = ev(n.operand)
            return ((~v) if n.op == "!" else (-v)), e
        op = n.op
        if op in LOGICAL:
            a, ea = ev(n.left)
            b, eb = ev(n.right)
            if op == "&&":
                err = _or(ea, None if eb is None else (eb & a))
                return a & b, err
            err = _or(ea, None if eb is None else (eb & ~a))
            return a | b, err
        a, ea = ev(n.left)
        b, eb = ev(n.right)
        err = _or(ea, eb)
        if op in COMPARISONS:
            if isinstance(a, Str) or isinstance(b, Str) or _is_str_var(n.left, var_types) \
                    or _is_str_var(n.right, var_types):
                a = _str_codes(n.left, a, strings_of)
                b = _str_codes(n.right, b, strings_of)
            r = _CMP[op](a, b)
            return (np.broadcast_to(r, (nrows,)) if np.ndim(r) == 0 else r), err
        if op in ("/", "%"):
            zero = np.asarray(b) == 0
            if np.ndim(zero) == 0:
                zero = np.full(nrows, bool(zero))
            err = _or(err, zero)
            a_f = _is_float(a)
            b_f = _is_float(b)
            safe_b = np.where(zero, 1, b)
            if a_f or b_f:
                af = np.asarray(a, dtype=np.float64)
                bf = np.asarray(safe_b, dtype=np.float64)
                return (af / bf if op == "/" else np.fmod(af, bf)), err
            ai = np.asarray(a, dtype=np.int64)
            bi = np.asarray(safe_b, dtype=np.int64)
            q = np.abs(ai) // np.abs(bi)
            q = np.where((ai < 0) != (bi < 0), -q, q)
            return (q if op == "/" else ai - q * bi), err
        if op == "^":
            if _is_float(a) or _is_float(b):
                return np.power(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)), err
            bi = np.asarray(b, dtype=np.int64)
            if np.any(bi < 0):
                raise NotVectorizable("negative exponent")
            return np.power(np.asarray(a, dtype=np.int64), bi), err
        if _is_float(a) or _is_float(b):
            a = np.asarray(a, dtype=np.float64)
            b = np.asarray(b, dtype=np.float64)
        return _ARITH[op](a, b), err

    val, err = ev(node)
    if np.ndim(val) == 0:
        val = np.full(nrows, val)
    return val, err


def _contains_str(n: Node) -> bool:
    if isinstance(n, Str):
        return True
    if isinstance(n, Unary):
        return _contains_str(n.operand)
    if isinstance(n, Binary):
        return _contains_str(n.left) or _contains_str(n.right)
    return False


def _contains_float(n: Node) -> bool:
    if isinstance(n, Num):
        return isinstance(n.value, float)
    if isinstance(n, Unary):
        return _contains_float(n.operand)
    if isinstance(n, Binary):
        return _contains_float(n.left) or _contains_float(n.right)
    return False


def _contains_pow(n: Node) -> bool:
    if isinstance(n, Unary):
        return _contains_pow(n.operand)
    if isinstance(n, Binary):
        return n.op == "^" or _contains_pow(n.left) or _contains_pow(n.right)
    return False


def _is_str_var(n: Node, var_types) -> bool:
    return isinstance(n, Var) and var_types.get(n.name) == "str"


def _str_codes(n: Node, v, strings_of):
    if isinstance(v, Str):
        return v.value
    if isinstance(n, Var) and n.name in strings_of:
        table = np.array(strings_of[n.name], dtype=object)
        return table[v]
    return v


def _is_float(x) -> bool:
    if isinstance(x, float):
        return True
    return isinstance(x, np.ndarray) and x.dtype.kind == "f"


def _or(a, b):
    if a is None:
        return b
    if b is None:
        return a
    return a | b


_CMP = {
    "==": lambda a, b: a == b,
    "!=": lambda a, b: a != b,
    "<": lambda a, b: a < b,
    "<=": lambda a, b: a <= b,
    ">": lambda a, b: a > b,
    ">=": lambda a, b: a >= b,
}
_ARITH = {
    "+": lambda a, b: a + b,
    "-": lambda a, b: a - b,
    "*": lambda a, b: a * b,
}
