"""Time a list of configurations of one problem (reference protocol, verified).

    python tools/run_configs.py hotspot "4,16,4,2,4,4,1;64,2,4,2,6,3,1" [--runs 7]
    python tools/run_configs.py hotspot --sample 200 --seed 1   # stratified sample
Prints one JSON line per configuration.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200.cuda_backend import CudaTarget  # noqa: E402
from paper_2407_11488_b200.measure import MeasurementProtocol  # noqa: E402
from paper_2407_11488_b200.paramspace import config_key  # noqa: E402
from paper_2407_11488_b200.problems import make_problem  # noqa: E402
from paper_2407_11488_b200.sweep import stratified_sample  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("problem")
ap.add_argument("configs", nargs="?", default="")
ap.add_argument("--runs", type=int, default=7)
ap.add_argument("--sample", type=int, default=0)
ap.add_argument("--param", default=None)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
prob = make_problem(a.problem)
cfgs = [tuple(int(x) for x in c.split(",")) for c in a.configs.split(";") if c.strip()]
if a.sample:
    cfgs += stratified_sample(prob.space, a.sample, a.seed, a.param)
tgt = CudaTarget(prob)
proto = MeasurementProtocol(warmup_runs=1, benchmark_runs=a.runs, flush_l2=True)
for i, c in enumerate(cfgs):
    if i % 8 == 0:
        tgt.prefetch(cfgs[i:])
    obs = tgt.execute(c, proto)
    tgt.collect_attrs()
    info = tgt.extras.get(config_key(c), {})
    mode = prob.kernel_mode(dict(zip(prob.space.param_names, c)))[0] if hasattr(prob, "kernel_mode") else None
    print(json.dumps({"config": list(c), "status": obs.status.value, "time_ms": obs.time_ms, "mode": mode,
                      "regs": info.get("regs"), "launch_ms": info.get("launch_ms"),
                      "detail": obs.detail[:200] if obs.detail else None}), flush=True)
