"""Where does a sweep's device time go besides the tuned kernels?

    python tools/sweep_gaps.py hotspot --n 40
Runs the same configurations (cubins precompiled, untimed) under protocol
variants and prints, per variant, configs/s and sweep efficiency
(sum of (1 warmup + 7 runs) x mean config time / device time between
stream markers): full protocol; no L2 flush; no verification; no module
preload; sequential execute instead of the pipeline.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200 import runtime as rt  # noqa: E402
from paper_2407_11488_b200.cuda_backend import CudaTarget  # noqa: E402
from paper_2407_11488_b200.measure import MeasurementProtocol  # noqa: E402
from paper_2407_11488_b200.problems import make_problem  # noqa: E402
from paper_2407_11488_b200.sweep import stratified_sample  # noqa: E402

PARAM = {"hotspot": "temporal_tiling_factor", "convolution": "block_size_x", "gemm": "MWG",
         "dedispersion": "block_size_x"}

ap = argparse.ArgumentParser()
ap.add_argument("problem")
ap.add_argument("--n", type=int, default=40)
a = ap.parse_args()
prob = make_problem(a.problem)
dev = rt.Device(0)
configs = stratified_sample(prob.space, a.n, 1, PARAM[a.problem])
for variant in ["full", "no_flush", "no_verify", "no_preload", "sequential", "full"]:
    tgt = CudaTarget(prob, device=dev, verify=variant != "no_verify")
    tgt.retire_cap = 1 << 14
    if variant == "no_preload":
        tgt.preload_depth = 0
    for c in configs:  # compile untimed
        tgt.compiler.compile(tgt.source_for(dict(zip(prob.space.param_names, c))),
                             prob.options(dict(zip(prob.space.param_names, c))))
    proto = MeasurementProtocol(warmup_runs=1, benchmark_runs=7, flush_l2=variant != "no_flush")
    dev.mark(0)
    t0 = time.perf_counter()
    if variant == "sequential":
        obs = []
        for i, c in enumerate(configs):
            if i % 4 == 0:
                tgt.prefetch(configs[i:])
            tgt.preload(configs[i + 1:])
            obs.append((c, tgt.execute(c, proto)))
    else:
        obs = list(tgt.execute_many(configs, proto))
    dev.mark(1)
    ms = dev.elapsed_ms(0, 1)
    wall = time.perf_counter() - t0
    kern = sum(8 * o.time_ms for _, o in obs if o.ok)
    host = {k: round(sum(tgt.extras.get(",".join(map(str, c)), {}).get(k, 0.0) for c, _ in obs), 4)
            for k in ("compile_wait_s", "t_load_s", "t_setup_s", "t_run_s")}
    print(json.dumps({"variant": variant, "configs_per_s": round(len(obs) / (ms / 1e3), 2),
                      "efficiency": round(kern / ms, 4), "device_ms": round(ms, 2), "wall_s": round(wall, 3),
                      "kernel_ms": round(kern, 2), "ok": sum(o.ok for _, o in obs), "host": host}), flush=True)
    tgt.close()
