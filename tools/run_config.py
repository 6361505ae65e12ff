"""Run ONE configuration of one problem a few times (ncu target).

    python tools/run_config.py hotspot 64,4,2,4,10,2,1 [--runs 3]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("TSG_LINEINFO", "1")  # source-level ncu pages

from paper_2407_11488_b200.cuda_backend import CudaTarget  # noqa: E402
from paper_2407_11488_b200.measure import MeasurementProtocol  # noqa: E402
from paper_2407_11488_b200.problems import make_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("problem")
ap.add_argument("config")
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--no-verify", action="store_true")
a = ap.parse_args()
prob = make_problem(a.problem)
cfg = tuple(int(x) for x in a.config.split(","))
assert prob.space.is_valid(cfg), cfg
tgt = CudaTarget(prob, verify=not a.no_verify)
obs = tgt.execute(cfg, MeasurementProtocol(warmup_runs=1, benchmark_runs=a.runs, flush_l2=True))
print(a.problem, cfg, obs.status.value, obs.time_ms, tgt.extras.get(a.config))
