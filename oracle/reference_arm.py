"""The reference's OWN CPU path, timed: unmodified tunescape + C kernel program.

BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): bench.py's
``--impl reference`` arm and its ``cpu_baseline`` leg call this, nothing
else does.

The reference (tunescape 0.1.0, pure Python) is installed UNMODIFIED under
``baseline/_ref`` (``baseline/install_reference.sh``: ``pip install
--no-deps --target baseline/_ref`` of a copy of /root/reference/pkg) and
travels to the GPU box with the repo snapshot.  Its only executor is the
command backend (`ts/measure.py:218-305`); its CPU path for a kernel is
therefore its tuning loop driving a CPU benchmark program -- here
``oracle/tsbench_cpu`` (kernels.c, all host threads, full BASELINE size),
which self-reports 1 warm-up + 7 ``TUNE_TIME_MS`` lines per launch, so the
reference spawns one process per configuration and keeps the last 7
(`measure.py:273-283`).  The search is the reference's ``random_search``
(`ts/strategies.py:148-192`) with its default protocol (1 + 7 runs, mean).

If the install is missing (a host that never ran the recipe), callers fall
back to ``oracle/reference_port.py`` and say so (``kind: "port"``).
"""

from __future__ import annotations

import importlib
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"
PROGRAM = ROOT / "oracle" / "tsbench_cpu"


def available() -> bool:
    return (REF_DIR / "tunescape" / "__init__.py").exists() and PROGRAM.exists()


def _tunescape():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    mod = importlib.import_module("tunescape")
    if not str(Path(mod.__file__)).startswith(str(REF_DIR)):
        raise RuntimeError(f"'tunescape' resolved to {mod.__file__}, not the baseline/_ref install")
    return mod


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def timed_random_search(kernel: str, budget: int, seed: int, threads: int | None = None) -> dict:
    """One reference ``random_search`` of ``budget`` configurations of the
    bundled ``kernel`` space, every configuration timed by the reference's
    command backend running ``tsbench_cpu``.  Returns wall seconds and the
    reference's own result."""
    ts = _tunescape()
    from tunescape.measure import MeasurementProtocol, command_backend
    from tunescape.paramspace import bundled_space
    from tunescape.strategies import random_search

    threads = threads or host_threads()
    space = bundled_space(kernel)
    slots = " ".join("{%s}" % n for n in space.param_names)
    backend = command_backend(f"{PROGRAM} {kernel} --threads {threads} --runs 8 {slots}")
    t0 = time.perf_counter()
    result = random_search(space, backend, MeasurementProtocol(), budget, seed)
    secs = time.perf_counter() - t0
    ok = [o for _, o in result.trace if o.ok]
    return {"configs": result.evaluations_used, "seconds": secs, "cores": threads,
            "ok": len(ok), "mean_kernel_ms": (sum(o.time_ms for o in ok) / len(ok)) if ok else None,
            "tunescape": getattr(ts, "__version__", "?"),
            "sample": (f"{result.evaluations_used} {kernel} configurations: unmodified reference "
                       f"(baseline/_ref tunescape) random_search, command backend -> oracle/tsbench_cpu "
                       f"(C kernel, {threads} threads, full size), 1 warmup + 7 runs each")}
