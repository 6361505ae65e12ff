"""Brute-force tune a whole bundled space on the GPU(s) and write its caches.

    python tools/full_sweep.py convolution --out profiles/round1/caches
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        tools/full_sweep.py convolution --out ...          (config sharding, N8)

The whole path of the reference's ``tunescape tune --strategy brute`` with
the in-process ``cuda`` backend: enumerate + restrict, NVRTC compile
(pipelined), load, 1 warmup + 7 timed runs with L2 flushes, on-device
verification, Observation, merged by enumeration index across ranks.
Writes the native cache and a Kernel-Tuner-format cache (the format the
reference's ``import_external_cache`` reads) and prints a JSON summary.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200 import runtime as rt  # noqa: E402
from paper_2407_11488_b200.cuda_backend import CudaTarget  # noqa: E402
from paper_2407_11488_b200.measure import MeasurementProtocol, cuda_backend  # noqa: E402
from paper_2407_11488_b200.multigpu import sharded_brute_force, torch_dist_plumbing  # noqa: E402
from paper_2407_11488_b200.problems import make_problem  # noqa: E402
from paper_2407_11488_b200.store import write_cache, write_kernel_tuner_cache  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("problem")
    ap.add_argument("--out", default="gpurun_out/caches")
    ap.add_argument("--chunk", type=int, default=16)
    ap.add_argument("--limit", type=int, default=0, help="first N configurations only (0 = all)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    store, gather, rank, world = torch_dist_plumbing()
    prob = make_problem(a.problem)
    dev = rt.Device(local)
    target = CudaTarget(prob, device=dev)
    backend = cuda_backend(target)
    proto = MeasurementProtocol(warmup_runs=1, benchmark_runs=7, flush_l2=True)
    configs = list(prob.space.enumerate_configs())
    if a.limit:
        configs = configs[: a.limit]
    t0 = time.perf_counter()
    result, cache, stats = sharded_brute_force(prob.space, backend, proto, chunk=a.chunk, store=store,
                                               gather=gather, rank=rank, device_name=dev.info["name"],
                                               configs=configs)
    wall = time.perf_counter() - t0
    target.close()
    if rank == 0:
        out = Path(a.out)
        out.mkdir(parents=True, exist_ok=True)
        write_cache(cache, out / f"{a.problem}.tunescape.json")
        write_kernel_tuner_cache(cache, out / f"{a.problem}.kerneltuner.json", space=prob.space)
        ok = [o for _, o in result.trace if o.ok]
        times = sorted(o.time_ms for o in ok)
        summary = {
            "problem": a.problem, "configs": len(result.trace), "ok": len(ok), "world": world,
            "wall_s": round(wall, 2), "configs_per_s": round(len(result.trace) / wall, 2),
            "best": list(result.best) if result.best else None,
            "best_ms": result.best_observation.time_ms if result.best_observation else None,
            "best_over_median": round(times[len(times) // 2] / times[0], 3) if times else None,
            "best_over_worst": round(times[-1] / times[0], 3) if times else None,
            "failed": {s: sum(1 for _, o in result.trace if not o.ok and o.status.value == s)
                       for s in {o.status.value for _, o in result.trace if not o.ok}},
            "per_rank": [vars(s) for s in stats],
        }
        print(json.dumps(summary))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
