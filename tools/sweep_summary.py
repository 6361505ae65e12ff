"""Summarise a whole-space sweep cache (native tunescape format).

    python tools/sweep_summary.py hotspot gpurun_out/caches/hotspot.tunescape.json [--wall-s S] [--out F]

Writes {problem, configs, ok, best, best_ms, median/worst, best_over_median,
best_over_worst, by_mode{n, best_ms, median_ms}} -- the per-kernel B200
column of the paper's Table 4.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200.problems import make_problem  # noqa: E402
from paper_2407_11488_b200.store import loads_cache  # noqa: E402


def mode_of(prob, cfg: dict) -> str:
    if hasattr(prob, "kernel_mode"):
        return prob.kernel_mode(cfg)[0]
    if hasattr(prob, "window_span"):
        if prob.window_span(cfg) is not None:
            return "window"
        return "staged" if prob.staged_stages(cfg) else "plain"
    return "all"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("problem")
    ap.add_argument("cache")
    ap.add_argument("--wall-s", type=float, default=None)
    ap.add_argument("--command", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    prob = make_problem(a.problem)
    names = prob.space.param_names
    cache = loads_cache(Path(a.cache).read_text())
    ok = cache.ok_records()
    times = {k: o.time_ms for k, o in ok.items()}
    best = min(times, key=times.get)
    worst = max(times, key=times.get)
    med = statistics.median(times.values())
    by = {}
    for k, t in times.items():
        cfg = dict(zip(names, (int(x) for x in k.split(","))))
        by.setdefault(mode_of(prob, cfg), []).append(t)
    doc = {"problem": a.problem, "configs": len(cache.records), "ok": len(ok),
           "best": [int(x) for x in best.split(",")], "best_ms": round(times[best], 6),
           "median_ms": round(med, 6), "worst_ms": round(times[worst], 6),
           "best_over_median": round(med / times[best], 3), "best_over_worst": round(times[worst] / times[best], 3),
           "by_mode": {m: {"n": len(v), "best_ms": round(min(v), 4), "median_ms": round(statistics.median(v), 4)}
                       for m, v in sorted(by.items())}}
    # the paper's Table 4 metric per kernel: GFLOP/s for
    # convolution / hotspot / GEMM, GB/s (4 B loaded per add) for dedispersion
    if hasattr(prob, "paper_bytes"):
        work, unit = prob.paper_bytes(), "GB/s"
    else:
        work, unit = prob.flops(), "GFLOP/s"
    perf = sorted(work / (t * 1e6) for t in times.values())
    doc["table4"] = {"unit": unit, "median": round(statistics.median(perf), 1), "maximum": round(perf[-1], 1),
                     "impact": round(perf[-1] / statistics.median(perf), 2)}
    if a.wall_s:
        doc["wall_s"] = round(a.wall_s)
        doc["configs_per_s"] = round(len(cache.records) / a.wall_s, 2)
    if a.command:
        doc["command"] = a.command
    text = json.dumps(doc)
    if a.out:
        Path(a.out).write_text(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
