"""Domain-decomposed hotspot 16384^2 (BASELINE configs[4]); run under torchrun.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/dd_hotspot_bench.py --config 32,16,3,2,6,6,1
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11488_b200.dd_hotspot import cuda_run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="32,16,3,2,6,6,1")
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--iterations", type=int, default=20)
ap.add_argument("--repeats", type=int, default=3)
ap.add_argument("--no-verify", action="store_true")
a = ap.parse_args()
r = cuda_run(tuple(int(x) for x in a.config.split(",")), a.size, a.size, a.iterations, a.repeats,
             not a.no_verify)
if int(os.environ.get("RANK", 0)) == 0:
    print(json.dumps(r))
