"""CPU baseline: the reference tuning loop restated over the C oracle.

TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference's only executor runs a benchmark *program* per run and
reads its ``TUNE_TIME_MS`` line (`pkg/src/tunescape/measure.py:218-305`)
under the default protocol of 1 warmup + 7 recorded runs, mean
(`measure.py:59-79`), sequentially over the configurations a strategy
yields (`strategies.py:117-141`).  This port keeps that loop shape --
sequential configurations, warmup runs discarded, per-run wall time,
``statistics.fmean`` -- but runs the benchmark in-process through the C
restatement of the kernel (``liboracle.so``, all host threads) instead
of spawning a process per run (which would only add ~2 ms per run,
SURVEY §3.1).  The kernel arithmetic does not depend on the tunables on
a CPU, so every configuration costs the same full-size evaluation.
"""

from __future__ import annotations

import statistics
import time

import numpy as np

from . import kernels_ffi as K


class _Workload:
    def __init__(self, name: str):
        from paper_2407_11488_b200.problems import make_problem

        self.name = name
        self.prob = make_problem(name)
        p = self.prob
        if name == "convolution":
            self.args = (p.buffers()[0].init,)
        elif name == "hotspot":
            self.temp, self.power = p.temperature(), p.power()
            self.out = np.empty(p.W * p.H, np.float32)
            self.scratch = np.empty_like(self.out)
        elif name == "dedispersion":
            self.args = (p.buffers()[0].init,)
        elif name == "gemm":
            self.a, self.b = p.a(), p.b()
            self.out = np.empty(p.M * p.N, np.float32)

    def run_once(self):
        p = self.prob
        L = K.lib()
        if self.name == "convolution":
            K.convolution(p, self.args[0])
        elif self.name == "hotspot":
            k = p.k
            L.oracle_hotspot(K._p(self.out), K._p(self.temp), K._p(self.power), p.W, p.H,
                             p.iterations, k["sdc"], k["rx1"], k["ry1"], k["rz1"], k["amb"],
                             K._p(self.scratch))
        elif self.name == "dedispersion":
            K.dedispersion(p)
        else:
            L.oracle_gemm(K._p(self.out), K._p(self.a), K._p(self.b), p.M, p.N, p.K)


def evaluate(work: _Workload, warmup: int, runs: int) -> dict:
    """One configuration through the reference protocol (times in ms)."""
    times = []
    for r in range(warmup + runs):
        t0 = time.perf_counter()
        work.run_once()
        dt = (time.perf_counter() - t0) * 1000.0
        if r >= warmup:
            times.append(dt)
    return {"status": "ok", "times_ms": times, "time_ms": statistics.fmean(times)}


def timed_sample(workload: str, configs: list, budget_s: float = 15.0, warmup: int = 1,
                 runs: int = 7) -> dict:
    """Evaluate configurations sequentially until ``budget_s`` is spent.

    At least one configuration is always evaluated.  Returns the number
    of configurations, the seconds they took, the thread count and a
    description of the sample.
    """
    work = _Workload(workload)
    K.lib()
    done = 0
    t0 = time.perf_counter()
    per = []
    for c in configs:
        r = evaluate(work, warmup, runs)
        per.append(r["time_ms"])
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    secs = time.perf_counter() - t0
    return {"configs": done, "seconds": secs, "cores": K.threads(),
            "mean_kernel_ms": statistics.fmean(per),
            "sample": (f"{done} {workload} configurations x (1 warmup + 7 runs) of the full-size "
                       f"C-oracle kernel, {K.threads()} threads, budget {budget_s:g}s")}
