"""Generate tests/golden/reference_golden.json FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package (``tunescape`` from
/root/reference/pkg/src) and records what it computes -- enumeration
order digests, fingerprints, expression values/errors, neighbourhoods,
strategy traces over simulated caches, canonical cache text -- so the
B200 build's parity tests run anywhere (the GPU box has no reference).
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from tunescape import expressions as ex  # noqa: E402
from tunescape.measure import MeasurementProtocol, Observation, Status, simulated_backend  # noqa: E402
from tunescape.paramspace import (  # noqa: E402
    ConstraintExpr,
    ParameterDef,
    SearchSpaceSpec,
    bundled_space,
    config_key,
)
from tunescape.store import TuningCache, dumps_cache  # noqa: E402
from tunescape.strategies import brute_force, greedy_local_search, random_search  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_golden.json"


def digest(configs) -> str:
    h = hashlib.sha256()
    for c in configs:
        h.update((config_key(c) + "\n").encode())
    return h.hexdigest()


def spaces():
    out = {}
    for name in ("convolution", "hotspot", "dedispersion", "gemm"):
        s = bundled_space(name)
        cfgs = list(s.enumerate_configs())
        rec = dict(cartesian=s.cartesian_size, valid=len(cfgs), first=config_key(cfgs[0]),
                   last=config_key(cfgs[-1]), digest=digest(cfgs), fingerprint=s.fingerprint(),
                   text=s.to_text())
        # neighbourhoods of a few fixed configurations
        rng = random.Random(name)
        picks = [cfgs[rng.randrange(len(cfgs))] for _ in range(5)]
        rec["neighbors"] = {config_key(c): [config_key(n) for n in s.neighbors(c)] for c in picks}
        rec["neighbors_adjacent"] = {config_key(c): [config_key(n) for n in s.neighbors(c, "adjacent")]
                                     for c in picks}
        if name == "hotspot":
            per_t = {}
            for c in cfgs:
                per_t[c[4]] = per_t.get(c[4], 0) + 1
            rec["per_temporal_tiling_factor"] = per_t
        out[name] = rec
    return out


_LEAVES = ["a", "b", "c", "0", "1", "2", "3", "7", "-5", "2.5", "0.5"]
_BIN = ["+", "-", "*", "/", "%", "^"]
_CMP = ["==", "!=", "<", "<=", ">", ">="]


def rand_arith(rng, depth):
    if depth == 0 or rng.random() < 0.3:
        return rng.choice(_LEAVES)
    if rng.random() < 0.15:
        return "-" + rand_arith(rng, depth - 1)
    s = f"{rand_arith(rng, depth - 1)} {rng.choice(_BIN)} {rand_arith(rng, depth - 1)}"
    return f"({s})" if rng.random() < 0.5 else s


def rand_bool(rng, depth):
    r = rng.random()
    if depth == 0 or r < 0.4:
        return f"{rand_arith(rng, 2)} {rng.choice(_CMP)} {rand_arith(rng, 2)}"
    if r < 0.55:
        return rng.choice(["!", "not "]) + "(" + rand_bool(rng, depth - 1) + ")"
    op = rng.choice(["&&", "||", "and", "or"])
    return f"{rand_bool(rng, depth - 1)} {op} {rand_bool(rng, depth - 1)}"


def expressions():
    rng = random.Random(1234)
    cases = []
    fixed = ["-7 / 2 == -3", "7 / -2 == -3", "-7 % 2 == -1", "7 % -2 == 1", "2 ^ 10 == 1024",
             "2 + 3 * 4 == 14", "-2 ^ 2 == -4", "(2 + 3) * 4 == 20", "10 / 4 == 2",
             "2 * 4096 ^ 3 == 137438953472", "2^3^2", "-2^-2", "2^-1", "a - - b * c ^ 2",
             "a ^ -b ^ c", "1.5e3 + .5 - 3e2", "x +", "((x)", "x $ y", "", "1 2", "x ==", "* 3",
             "a < b < c", "(a < b < c)", "!a", "a && b", "(a < 1) + 1", "mode == 1",
             "mode < 'x'", "mode == 'fast'", "z == 1", "3 / 0", "a % 0 == 1", "1 / 2.0"]
    srcs = fixed + [rand_bool(rng, 3) for _ in range(300)] + [rand_arith(rng, 4) for _ in range(200)]
    types = {"a": "int", "b": "int", "c": "int", "mode": "str", "x": "int"}
    envs = [dict(a=a, b=b, c=c, mode="fast", x=1) for a, b, c in
            [(1, 2, 3), (-4, 3, 2), (7, -2, 0), (0, 5, -3), (12, 4, 1)]]
    for src in srcs:
        rec = {"source": src}
        try:
            node = ex.parse_expression(src)
            rec["ast"] = repr(node)
        except Exception as e:  # noqa: BLE001
            rec["parse_error"] = [type(e).__name__, str(e)]
            cases.append(rec)
            continue
        try:
            rec["type"] = ex.check_types(node, types, src)
        except Exception as e:  # noqa: BLE001
            rec["type_error"] = [type(e).__name__, str(e)]
            cases.append(rec)
            continue
        vals = []
        for env in envs:
            try:
                v = ex.evaluate(node, env)
                vals.append(["ok", repr(v)])
            except Exception as e:  # noqa: BLE001
                vals.append(["err", type(e).__name__])
        rec["values"] = vals
        cases.append(rec)
    return cases


_POOL = ("{a} * {b} <= {cap}", "{a} % {b} == 0", "{a} <= {b}", "{a} + {b} >= {low}",
         "{a} == {v} || {b} != {v}", "({a} - {b}) / 2 != 1", "!({a} == {v})")


def random_space(rng, kernel):
    n_params = rng.randint(2, 5)
    params = {}
    for i in range(n_params):
        nv = rng.randint(2, 7)
        start, step = rng.randint(1, 4), rng.randint(1, 4)
        params[f"p{i}"] = [start + step * j for j in range(nv)]
    names = list(params)
    cons = []
    for _ in range(rng.randint(0, 3)):
        a, b = rng.sample(names, 2)
        cons.append(rng.choice(_POOL).format(a=a, b=b, cap=rng.choice([16, 64, 256]),
                                             low=rng.randint(2, 8), v=rng.choice(params[a])))
    parameters = tuple(ParameterDef(n, tuple(v)) for n, v in params.items())
    return SearchSpaceSpec(kernel_name=kernel, parameters=parameters,
                           constraints=tuple(ConstraintExpr.parse(c, parameters) for c in cons))


def strategies():
    rng = random.Random(99)
    out = []
    proto = MeasurementProtocol()
    for i in range(12):
        s = random_space(rng, f"rand{i}")
        cfgs = list(s.enumerate_configs())
        if not cfgs:
            continue
        records = {}
        for c in cfgs:
            if rng.random() < 0.1:
                records[config_key(c)] = Observation(Status(rng.choice(["compile_failed", "invalid"])))
            else:
                t = round(rng.uniform(0.1, 100.0), 6)
                records[config_key(c)] = Observation(Status.OK, (t,), t, s.metric_value(t, c))
        cache = TuningCache(kernel_name=s.kernel_name, device_name="devA",
                            param_order=s.param_names, records=records,
                            space_fingerprint=s.fingerprint())
        be = simulated_backend(cache)
        rec = {"text": s.to_text(), "valid": [config_key(c) for c in cfgs],
               "records": {k: [o.status.value, o.time_ms] for k, o in records.items()}}
        bf, bf_cache = brute_force(s, be, proto)
        rec["brute_best"] = config_key(bf.best) if bf.best else None
        rec["cache_text"] = dumps_cache(bf_cache)
        runs = []
        for seed in (0, 1, 7):
            for budget in (1, 5, len(cfgs) + 3):
                r = random_search(s, be, proto, budget=budget, seed=seed)
                runs.append(dict(kind="random", seed=seed, budget=budget,
                                 trace=[config_key(c) for c, _ in r.trace], notes=list(r.notes),
                                 best=config_key(r.best) if r.best else None))
                g = greedy_local_search(s, be, proto, budget=budget, seed=seed)
                runs.append(dict(kind="greedy", seed=seed, budget=budget,
                                 trace=[config_key(c) for c, _ in g.trace], notes=list(g.notes),
                                 best=config_key(g.best) if g.best else None,
                                 segments=[[list(map(config_key, sg.path)), sg.reached_minimum]
                                           for sg in g.segments]))
                g2 = greedy_local_search(s, be, proto, budget=budget, seed=seed,
                                         first_improvement=True, scheme="adjacent")
                runs.append(dict(kind="greedy_first_adjacent", seed=seed, budget=budget,
                                 trace=[config_key(c) for c, _ in g2.trace], notes=list(g2.notes),
                                 best=config_key(g2.best) if g2.best else None))
        rec["runs"] = runs
        out.append(rec)
    return out


def main():
    doc = {"generator": "tests/golden/make_golden.py", "reference": str(REF),
           "spaces": spaces(), "expressions": expressions(), "strategies": strategies()}
    # metric known answers (ref tests/test_measure.py:222-225)
    g = bundled_space("gemm")
    c = next(iter(g.enumerate_configs()))
    doc["metric"] = {"gemm_6.939": g.metric_value(6.939, c),
                     "conv_1.0": bundled_space("convolution").metric_value(1.0, next(iter(
                         bundled_space("convolution").enumerate_configs())))}
    OUT.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
