"""``cmd:`` backend program: lets the UNMODIFIED reference CLI drive B200.

The reference's command backend runs a program per configuration and
reads ``TUNE_TIME_MS <float>`` lines from stdout; when the first launch
prints several lines it treats the program as self-reporting and keeps
the last ``benchmark_runs`` (`pkg/src/tunescape/measure.py:218-305`,
contract in `pkg/README.md:107-121`).  On failure the program exits
non-zero and may print ``TUNE_STATUS compile_failed|runtime_failed|
invalid`` (`measure.py:206-215`).

Usage with the reference (template placeholders filled by tunescape)::

    tunescape tune --space hotspot --strategy random --budget 8 \\
      --backend 'cmd:python -m paper_2407_11488_b200.tsbench --kernel hotspot \\
                 --config {block_size_x},{block_size_y},{tile_size_x},{tile_size_y},\\
{temporal_tiling_factor},{loop_unroll_factor_t},{sh_power}'

Each invocation creates a CUDA context and uploads the problem, so this
route costs ~seconds per configuration: it exists for interop and
parity, the in-process ``cuda`` backend is the throughput path.
"""

from __future__ import annotations

import argparse
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tsbench")
    ap.add_argument("--kernel", required=True, choices=["convolution", "hotspot", "dedispersion", "gemm"])
    ap.add_argument("--config", required=True, help="comma-separated values in space order")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--runs", type=int, default=7)
    ap.add_argument("--size", default=None, help="problem override, e.g. width=512,height=512")
    ap.add_argument("--no-verify", action="store_true")
    a = ap.parse_args(argv)

    from .cuda_backend import CudaTarget
    from .measure import MeasurementProtocol, Status
    from .problems import make_problem

    kw = {}
    if a.size:
        for part in a.size.split(","):
            k, v = part.split("=")
            kw[k] = int(v) if v.lstrip("-").isdigit() else float(v)
    prob = make_problem(a.kernel, **kw)
    config = prob.space.config_from_key(a.config)
    if not prob.space.is_valid(config):
        print("TUNE_STATUS invalid")
        return 3
    target = CudaTarget(prob, verify=not a.no_verify)
    obs = target.execute(config, MeasurementProtocol(warmup_runs=0, benchmark_runs=a.warmup + a.runs))
    if obs.status is not Status.OK:
        print(f"TUNE_STATUS {obs.status.value}")
        print(obs.detail or "", file=sys.stderr)
        return 2
    # self-reporting: warmup lines first, the reference keeps the last `runs`
    for t in obs.times_ms:
        print(f"TUNE_TIME_MS {t:.6f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
